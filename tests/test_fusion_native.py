"""The native plan_spatial_fusion port (csrc/fusion_plan.cpp) reproduces the
unmodified reference planner's FusionPlan (fusion.py:108-220) exactly:
groups, memory_bytes and saved_bytes, including a budget-binding case."""
import json

import numpy as np
import pytest

from paper_2309_03523_b200.plan import PlanArrays, native_fusion


def _pa(z, prof):
    return PlanArrays(T=0, feature_dim=16, inst_entity=z["inst_entity"], inst_t=z["inst_t"],
                      spatial_edges=z["spatial_edges"], temporal_links=z["temporal_links"],
                      structure_device=z["structure_device"], chunk_of=z["chunk_of"],
                      n_devices=len(z["queue_ptr"]) - 1, profile=prof)


@pytest.mark.parametrize("name", ["f6k_d2", "f6k_d2_tight", "f8k_d1_lstm", "f30k_d3"])
def test_native_fusion_equals_reference(golden_dir, name):
    z = np.load(golden_dir / f"fusion_{name}.npz")
    meta = json.loads(bytes(z["meta"]).decode())
    qp, qc = z["queue_ptr"], z["queue_chunks"]
    queues = [qc[qp[d]:qp[d + 1]] for d in range(len(qp) - 1)]
    gd, gp, gc, mem, sav = native_fusion(_pa(z, meta["profile"]), queues, meta["budget"])
    np.testing.assert_array_equal(gd, z["group_device"])
    np.testing.assert_array_equal(gp, z["group_ptr"])
    np.testing.assert_array_equal(gc, z["group_chunks"])
    np.testing.assert_array_equal(mem, z["group_memory"])
    np.testing.assert_array_equal(sav, z["group_saved"])


def test_native_fusion_equals_reference_c1_artifacts(artifacts_dir):
    d = artifacts_dir / "c1"
    from paper_2309_03523_b200.plan import load_plan_npz
    pa = load_plan_npz(d / "plan.npz")
    z = np.load(d / "plan.npz")
    queues = [z["queue_chunks"][z["queue_ptr"][i]:z["queue_ptr"][i + 1]] for i in range(4)]
    gd, gp, gc, mem, sav = native_fusion(pa, queues)
    fus = json.loads((d / "fusion.json").read_text())
    ref = [(int(dv), g) for dv, gl in sorted((int(k), v) for k, v in fus["devices"].items()) for g in gl]
    assert len(ref) == len(gd)
    for i, (dv, g) in enumerate(ref):
        assert gd[i] == dv
        assert list(gc[gp[i]:gp[i + 1]]) == g["chunks"]
        assert mem[i] == g["memory_bytes"] and sav[i] == g["saved_bytes"]


def test_native_fusion_budget_exceeded(golden_dir):
    z = np.load(golden_dir / "fusion_f6k_d2.npz")
    meta = json.loads(bytes(z["meta"]).decode())
    queues = [z["queue_chunks"][z["queue_ptr"][0]:z["queue_ptr"][1]]]
    with pytest.raises(ValueError, match="BudgetExceededError"):
        native_fusion(_pa(z, meta["profile"]), queues, memory_budget=1000)


@pytest.mark.parametrize("name", ["f6k_d2", "f30k_d3"])
def test_heap_path_equals_component_fast_path(golden_dir, name, monkeypatch):
    """The general greedy heap path and the non-binding connected-component
    shortcut give identical plans (and both equal the reference)."""
    z = np.load(golden_dir / f"fusion_{name}.npz")
    meta = json.loads(bytes(z["meta"]).decode())
    qp, qc = z["queue_ptr"], z["queue_chunks"]
    queues = [qc[qp[d]:qp[d + 1]] for d in range(len(qp) - 1)]
    fast = native_fusion(_pa(z, meta["profile"]), queues, meta["budget"])
    monkeypatch.setenv("DGC_FUSION_FORCE_HEAP", "1")
    heap = native_fusion(_pa(z, meta["profile"]), queues, meta["budget"])
    for a, b in zip(fast, heap):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(heap[2], z["group_chunks"])
