"""Build the benchmark graphs and DGC plans with the UNMODIFIED reference
planner (``dynpart``, imported read-only from /root/reference) and freeze them
as compact artifacts the GPU box can load without the reference.

The plan is consumed unchanged: this script is
the only place the reference planner runs; the product only reads its output.

Usage (in the build container only):
    PYTHONPATH=/root/reference/pkg/src python tools/make_artifacts.py c1 [c2 ...]
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

import dynpart
from dynpart import graphstore, sim
from dynpart.costmodel import ModelProfile
from dynpart.cli import _write_json
from dynpart.partition import chunk_graph_to_json

ROOT = Path(__file__).resolve().parents[1]

# SURVEY.md §8(d) / BASELINE.md §3 synthetic specs
CONFIGS = {
    "c1": dict(N=10_000, T=16, sigma_mult=1.0, D=4, F=16,
               profile=ModelProfile(1, 2, 1, "previous-only", 16, 4), fuse=True),
    # fusion "native": build_plan(fuse=False) by the reference, then the
    # bit-exact native plan_spatial_fusion port (tests/test_fusion_native.py):
    # the reference's Python fusion planner ran > 86 CPU-min and 46 GB at 200k
    "c2": dict(N=200_000, T=32, sigma_mult=1.0, D=1, F=16,
               profile=ModelProfile(1, 2, 2, "previous-only", 16, 4), fuse="native"),
    # the C2 graph re-planned for 2/4/8 devices (strong-scaling runs); fusion
    # off: numerics are fusion-invariant and the Python
    # fusion planner does not finish at this size in useful time
    "c2d2": dict(N=200_000, T=32, sigma_mult=1.0, D=2, F=16,
                 profile=ModelProfile(1, 2, 2, "previous-only", 16, 4), fuse=False),
    "c2d4": dict(N=200_000, T=32, sigma_mult=1.0, D=4, F=16,
                 profile=ModelProfile(1, 2, 2, "previous-only", 16, 4), fuse=False),
    "c2d8": dict(N=200_000, T=32, sigma_mult=1.0, D=8, F=16,
                 profile=ModelProfile(1, 2, 2, "previous-only", 16, 4), fuse=False),
    # C3: EvolveGCN-style profile ModelProfile(1,2,0): no vertex-level temporal
    # messages, so chunks are snapshot-local
    "c3d2": dict(N=1_000_000, T=64, sigma_mult=1.0, D=2, F=16,
                 profile=ModelProfile(1, 2, 0, "previous-only", 16, 4), fuse="native"),
    "c3d4": dict(N=1_000_000, T=64, sigma_mult=1.0, D=4, F=16,
                 profile=ModelProfile(1, 2, 0, "previous-only", 16, 4), fuse="native"),
    "c3d8": dict(N=1_000_000, T=64, sigma_mult=1.0, D=8, F=16,
                 profile=ModelProfile(1, 2, 0, "previous-only", 16, 4), fuse="native"),
    # C4: the C3 graph on 8 devices planned with the GCN+GRU recurrent profile
    # (an EvolveGCN plan is snapshot-local and cuts almost
    # nothing); the staleness sweep runs on it (tools/stale_sweep.py --plan c4d8)
    "c4d8": dict(N=1_000_000, T=64, sigma_mult=1.0, D=8, F=16,
                 profile=ModelProfile.recurrent(16), fuse=False, native_propagate=True),
    # C5: 10M instances x 128 snapshots, sigma = 2 mu, EvolveGCN profile, D = 8.
    # PGC through the native bit-exact propagate port (the Python label
    # propagation needs hours at 10M); assignment by the reference; fusion off
    # (numerics are fusion-invariant)
    "c5d8": dict(N=10_000_000, T=128, sigma_mult=2.0, D=8, F=16,
                 profile=ModelProfile(1, 2, 0, "previous-only", 16, 4), fuse=False,
                 native_propagate=True, native_generate=True),
    # small EvolveGCN plans for the parity tests
    "e2": dict(N=3_000, T=8, sigma_mult=1.0, D=2, F=16,
               profile=ModelProfile(1, 2, 0, "previous-only", 16, 4), fuse=True),
    # small multi-device variants used by the parity tests (fast to plan)
    "t2": dict(N=3_000, T=8, sigma_mult=1.0, D=2, F=16,
               profile=ModelProfile(1, 2, 1, "previous-only", 16, 4), fuse=True),
    "t4": dict(N=4_000, T=8, sigma_mult=1.0, D=4, F=16,
               profile=ModelProfile(1, 2, 2, "previous-only", 16, 4), fuse=True),
}


def spec_for(cfg: dict) -> graphstore.SyntheticSpec:
    N, T = cfg["N"], cfg["T"]
    E = 4 * N
    mu = E / T
    return graphstore.SyntheticSpec(
        total_vertices=N, total_edges=E, T=T,
        edges_per_snapshot_mean=mu, edges_per_snapshot_stddev=cfg["sigma_mult"] * mu,
        presence_length_distribution=graphstore.LengthDistribution.bimodal(
            1, max(1, T // 4), max(1, T // 2), T, 0.2),
        rng_seed=0, feature_dim=cfg["F"], edge_attachment="preferential")


def build(name: str) -> None:
    cfg = CONFIGS[name]
    out = ROOT / "artifacts" / name
    out.mkdir(parents=True, exist_ok=True)
    t0 = time.time()
    if cfg.get("native_generate"):
        # the native generator (csrc/generate.cpp): seconds
        # instead of ~25 min; the reference DynamicGraph validates its output
        sys.path.insert(0, str(ROOT))
        from paper_2309_03523_b200.generate import generate as native_generate
        g = native_generate(spec_for(cfg)).to_dynamic_graph()
    else:
        g = graphstore.generate(spec_for(cfg))
    t1 = time.time()
    cluster = sim.ClusterSpec(n_devices=cfg["D"])
    if cfg.get("native_propagate"):
        sys.path.insert(0, str(ROOT))
        from paper_2309_03523_b200.partition import native_planner
        with native_planner():
            plan = sim.build_plan(g, "pgc", cfg["profile"], cluster, fuse=cfg["fuse"] is True)
    else:
        plan = sim.build_plan(g, "pgc", cfg["profile"], cluster, fuse=cfg["fuse"] is True)
    t2 = time.time()
    print(f"[{name}] generate {t1 - t0:.1f}s build_plan {t2 - t1:.1f}s "
          f"chunks={len(plan.chunk_graph.chunks)}", flush=True)

    inst = np.asarray(g.instances, dtype=np.int64).reshape(-1, 2)
    chunk_of = np.empty(g.n_instances, dtype=np.int64)
    for c in plan.chunk_graph.chunks:
        for v in c.members:
            chunk_of[g.index_of(v)] = c.id
    queues = plan.assignment.queues
    groups = []  # (device, [chunk ids]) in FusionPlan order
    fusion_src = None
    if plan.fusion is not None:
        fusion_src = "reference plan_fusion"
        for dev, gl in sorted(plan.fusion.groups_by_device.items()):
            for grp in gl:
                groups.append((dev, list(grp.chunk_ids)))
    elif cfg["fuse"] == "native":
        sys.path.insert(0, str(ROOT))
        from paper_2309_03523_b200.plan import PlanArrays, native_fusion
        pa = PlanArrays(T=g.T, feature_dim=g.feature_dim,
                        inst_entity=inst[:, 0].astype(np.int32), inst_t=inst[:, 1].astype(np.int32),
                        spatial_edges=g.spatial_edge_index().astype(np.int32),
                        temporal_links=g.temporal_link_index().astype(np.int32),
                        structure_device=plan.structure_device.astype(np.int32),
                        chunk_of=chunk_of.astype(np.int32), n_devices=cfg["D"],
                        profile=cfg["profile"].to_dict())
        t3 = time.time()
        gd, gp, gc, _, _ = native_fusion(pa, queues, cluster.memory_budget)
        print(f"[{name}] native fusion {time.time() - t3:.1f}s groups={len(gd)}", flush=True)
        for i in range(len(gd)):
            groups.append((int(gd[i]), [int(c) for c in gc[gp[i]:gp[i + 1]]]))
        fusion_src = "native bit-exact port of plan_spatial_fusion (csrc/fusion_plan.cpp)"
    meta = {
        "name": name, "T": g.T, "feature_dim": g.feature_dim,
        "n_instances": g.n_instances, "n_spatial_edges": g.n_spatial_edges,
        "n_devices": cfg["D"], "profile": cfg["profile"].to_dict(),
        "fused": bool(groups), "fusion_source": fusion_src,
        "generate_s": t1 - t0, "build_plan_s": t2 - t1,
        "generator": "native (csrc/generate.cpp)" if cfg.get("native_generate") else "reference",
        "reference": "dynpart " + dynpart.__version__,
    }
    np.savez_compressed(
        out / "plan.npz",
        meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8),
        inst_entity=inst[:, 0].astype(np.int32), inst_t=inst[:, 1].astype(np.int32),
        spatial_edges=g.spatial_edge_index().astype(np.int32),
        temporal_links=g.temporal_link_index().astype(np.int32),
        structure_device=plan.structure_device.astype(np.int32),
        chunk_of=chunk_of.astype(np.int32),
        queue_ptr=np.cumsum([0] + [len(q) for q in queues]).astype(np.int64),
        queue_chunks=np.asarray([c for q in queues for c in q], dtype=np.int32),
        group_device=np.asarray([d for d, _ in groups], dtype=np.int32),
        group_ptr=np.cumsum([0] + [len(c) for _, c in groups]).astype(np.int64),
        group_chunks=np.asarray([c for _, cs in groups for c in cs], dtype=np.int32),
    )
    if g.n_instances <= 20_000:
        # the reference's own stage artifacts (cli.py:27-33) for the loader tests
        graphstore.save_graph(g, str(out / "graph.dg"))
        _write_json(out / "chunks.json", chunk_graph_to_json(plan.chunk_graph, cfg["profile"]))
        _write_json(out / "assignment.json", {**plan.assignment.to_dict(), "method": "pgc"})
        if plan.fusion is not None:
            _write_json(out / "fusion.json", plan.fusion.to_dict())
    print(f"[{name}] wrote {out}", flush=True)




def share_graphs(groups=(("c2", ("c2", "c2d2", "c2d4", "c2d8")), ("c3", ("c3d2", "c3d4", "c3d8", "c4d8")),
                         ("c5", ("c5d8",)))):
    """Plans of one graph share artifacts/<g>_graph.npz (the graph arrays); each
    plan.npz keeps only the plan arrays and names its graph file in meta."""
    import hashlib
    gkeys = ["inst_entity", "inst_t", "spatial_edges", "temporal_links"]
    for gname, members in groups:
        ref = None
        for m in members:
            p = ROOT / "artifacts" / m / "plan.npz"
            if not p.exists():
                continue
            z = dict(np.load(p))
            if "inst_entity" not in z:
                continue  # already split
            h = hashlib.sha1(b"".join(z[k].tobytes() for k in gkeys)).hexdigest()
            if ref is None:
                ref = h
                np.savez_compressed(ROOT / "artifacts" / f"{gname}_graph.npz", **{k: z[k] for k in gkeys})
            assert h == ref, (m, "graph differs")
            meta = json.loads(bytes(z["meta"]).decode())
            meta.update(graph_npz=f"{gname}_graph.npz", graph_sha1=h)
            rest = {k: v for k, v in z.items() if k not in gkeys and k != "meta"}
            np.savez_compressed(p, meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8), **rest)


if __name__ == "__main__":
    for n in sys.argv[1:]:
        build(n)
    share_graphs()
