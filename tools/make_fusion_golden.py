"""Golden FusionPlans from the UNMODIFIED reference planner (fusion.py) for the
native port's tests: graphs of a few sizes/budgets. Run in the build container:
PYTHONPATH=/root/reference/pkg/src python tools/make_fusion_golden.py"""
import json
import time
from pathlib import Path

import numpy as np

from dynpart import graphstore, sim
from dynpart.costmodel import ModelProfile
from dynpart.fusion import MemCoeffs

ROOT = Path(__file__).resolve().parents[1]
cases = [  # (name, N, T, D, profile, budget)
    ("f6k_d2", 6000, 12, 2, ModelProfile(1, 2, 1, "previous-only", 16, 4), 1 << 30),
    ("f6k_d2_tight", 6000, 12, 2, ModelProfile(1, 2, 1, "previous-only", 16, 4), 1_500_000),
    ("f8k_d1_lstm", 8000, 16, 1, ModelProfile(1, 2, 2, "previous-only", 16, 4), 1 << 30),
    ("f30k_d3", 30000, 24, 3, ModelProfile(1, 2, 1, "previous-only", 16, 4), 1 << 30),
]
out = {}
for name, N, T, D, prof, budget in cases:
    E = 4 * N
    spec = graphstore.SyntheticSpec(N, E, T, E / T, E / T,
                                    graphstore.LengthDistribution.bimodal(1, T // 4, T // 2, T, 0.2),
                                    rng_seed=3, feature_dim=16, edge_attachment="preferential")
    g = graphstore.generate(spec)
    t0 = time.time()
    plan = sim.build_plan(g, "pgc", prof, sim.ClusterSpec(n_devices=D, memory_budget=budget))
    dt = time.time() - t0
    inst = np.asarray(g.instances, dtype=np.int64).reshape(-1, 2)
    chunk_of = np.empty(g.n_instances, np.int64)
    for c in plan.chunk_graph.chunks:
        for v in c.members:
            chunk_of[g.index_of(v)] = c.id
    groups = [(d, list(gr.chunk_ids), gr.memory_bytes, gr.saved_bytes)
              for d, gl in sorted(plan.fusion.groups_by_device.items()) for gr in gl]
    np.savez_compressed(
        ROOT / "tests" / "golden" / f"fusion_{name}.npz",
        meta=np.frombuffer(json.dumps({"profile": prof.to_dict(), "budget": budget, "D": D,
                                       "T": T, "build_plan_s": dt}).encode(), dtype=np.uint8),
        inst_entity=inst[:, 0].astype(np.int32), inst_t=inst[:, 1].astype(np.int32),
        spatial_edges=g.spatial_edge_index().astype(np.int32),
        temporal_links=g.temporal_link_index().astype(np.int32),
        structure_device=plan.structure_device.astype(np.int32), chunk_of=chunk_of.astype(np.int32),
        queue_ptr=np.cumsum([0] + [len(q) for q in plan.assignment.queues]),
        queue_chunks=np.asarray([c for q in plan.assignment.queues for c in q], np.int32),
        group_device=np.asarray([d for d, *_ in groups], np.int32),
        group_ptr=np.cumsum([0] + [len(c) for _, c, *_ in groups]),
        group_chunks=np.asarray([c for _, cs, *_ in groups for c in cs], np.int32),
        group_memory=np.asarray([m for *_, m, _ in groups], np.int64),
        group_saved=np.asarray([s for *_, s in groups], np.int64))
    print(name, "groups", len(groups), "build_plan", round(dt, 1), "s", flush=True)
