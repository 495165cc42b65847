"""The native plan->layout builder (C ABI dgc_layout_build) equals the
independent Python restatement in oracle/layout.py, array by array; the three
plan loaders agree; native packing equals the reference golden vectors."""
import json

import numpy as np
import pytest

from oracle.layout import build_layouts
from paper_2309_03523_b200.layout import build_layout, pack_sequences_native
from paper_2309_03523_b200.plan import from_reference_artifacts, load_plan_npz

CMP = ["own_gid", "halo_gid", "group_ptr", "row_ptr", "col", "t_row_ptr", "t_col", "key_rows",
       "send_ptr", "send_pos", "recv_ptr", "recv_slot", "run_ptr", "run_rows", "run_pred_gid",
       "run_carry", "slot_row", "slot_mask", "slot_carry", "tkey_rows", "tsend_ptr", "tsend_pos",
       "trecv_ptr", "trecv_carry"]


@pytest.mark.parametrize("name", ["t2", "t4", "c1"])
def test_native_layout_matches_oracle(artifacts_dir, name):
    pa = load_plan_npz(artifacts_dir / name / "plan.npz")
    ref = build_layouts(pa.n_instances, pa.inst_entity, pa.inst_t, pa.spatial_edges,
                        pa.temporal_links, pa.structure_device, pa.chunk_of, pa.n_devices,
                        pa.group_device, pa.group_ptr, pa.group_chunks)
    for d in range(pa.n_devices):
        lay = build_layout(pa, d)
        for f in CMP:
            np.testing.assert_array_equal(lay.arrays[f], getattr(ref[d], f), err_msg=f"{name} d={d} {f}")
        np.testing.assert_allclose(lay.dinv, ref[d].dinv, rtol=0, atol=0)
        assert lay.padding == ref[d].padding and lay.naive_padding == ref[d].naive_padding


def test_loaders_agree_and_billing_inputs(artifacts_dir, golden_dir):
    a = load_plan_npz(artifacts_dir / "c1" / "plan.npz")
    b = from_reference_artifacts(artifacts_dir / "c1")
    for f in ("inst_entity", "inst_t", "spatial_edges", "temporal_links", "structure_device",
              "chunk_of", "group_device", "group_ptr", "group_chunks"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)
    z = np.load(golden_dir / "sim_c1.npz")
    lays = [build_layout(a, d) for d in range(a.n_devices)]
    # padding equals the reference's packed_padding per device (sim.py:492-500)
    assert sum(l.padding for l in lays) == z["rep_padding_slots"][0]
    assert sum(l.naive_padding for l in lays) == z["rep_naive_padding_slots"][0]
    # loaded rows x F x s equals the reference's loading_bytes (sim.py:487)
    prof = a.profile
    assert sum(l.loaded_rows for l in lays) * a.feature_dim * prof["bytes_per_scalar"] == z["rep_loading_bytes"][0]
    # cut spatial messages sourced per key sum to the reference's cut spatial count
    cut = z["cut"] & z["msg_spatial"]
    assert sum(int(l.key_ncut.sum()) for l in lays) == int(cut.sum())
    # temporal keys = sources of cut temporal messages
    tcut = z["cut"] & ~z["msg_spatial"]
    assert sum(len(l.tkey_rows) for l in lays) == int(tcut.sum())


def test_native_pack_matches_reference_golden(golden_dir):
    z = np.load(golden_dir / "packing.npz")
    ptr, meta = z["len_ptr"], z["meta"]
    roff = 0
    for i in range(len(meta)):
        lengths = z["lengths"][ptr[i]:ptr[i + 1]]
        R, L, pad, _ = meta[i]
        seq, pos, mask, padding = pack_sequences_native(lengths)
        rows = z["rows"][roff:roff + R * L].reshape(R, L, 2)
        np.testing.assert_array_equal(seq, rows[..., 0])
        np.testing.assert_array_equal(pos, rows[..., 1])
        np.testing.assert_array_equal(mask.reshape(-1), z["mask"][roff:roff + R * L])
        assert padding == pad
        roff += R * L


def test_plan_mismatch_raises(artifacts_dir):
    from paper_2309_03523_b200.plan import PlanGraphMismatch
    pa = load_plan_npz(artifacts_dir / "t2" / "plan.npz")
    pa.structure_device = pa.structure_device[:-1]
    with pytest.raises(PlanGraphMismatch):
        build_layout(pa, 0)
