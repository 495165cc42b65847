"""Golden PGC labels from the UNMODIFIED reference (dynpart.partition.propagate,
partition.py:200-270) for the native port's tests: the C1 graph plus generated
graphs covering the recurrent / LSTM / EvolveGCN (zero temporal weight) /
attention (all-snapshots fanout) profiles and binding size caps. Run in the
build container:
PYTHONPATH=/root/reference/pkg/src python tools/make_propagate_golden.py"""
import time
from pathlib import Path

import numpy as np

from dynpart import graphstore
from dynpart.costmodel import ModelProfile, edge_traffic
from dynpart.partition import _temporal_link_weights, default_size_cap, propagate

ROOT = Path(__file__).resolve().parents[1]


def chunk_of(g, cg):
    """Chunk id of every instance (ids = rank of the final label in np.unique,
    partition.py:298), so equal arrays mean equal labels up to their values'
    order -- exactly what _build_chunk_graph consumes."""
    out = np.empty(g.n_instances, np.int64)
    for c in cg.chunks:
        out[[g.index_of(v) for v in c.members]] = c.id
    return out


cases = []
g1 = graphstore.load_graph(ROOT / "artifacts" / "c1" / "graph.dg")
cases.append(("c1_recurrent", g1, ModelProfile.recurrent(16), default_size_cap(g1, 4)))
for name, N, T, prof, cap, seed, attach in [
    ("g3k_lstm", 3000, 10, ModelProfile(1, 2, 2, "previous-only", 16, 4), None, 1, "preferential"),
    ("g3k_evolve", 3000, 10, ModelProfile(1, 2, 0, "previous-only", 16, 4), None, 2, "preferential"),
    ("g2k_attention", 2000, 8, ModelProfile.attention(16), None, 3, "uniform"),
    ("g2k_cap3", 2000, 8, ModelProfile.recurrent(16), 3, 4, "preferential"),
    ("g4k_cap40", 4000, 12, ModelProfile.recurrent(16), 40, 5, "uniform"),
]:
    E = 4 * N
    spec = graphstore.SyntheticSpec(N, E, T, E / T, E / T,
                                    graphstore.LengthDistribution.bimodal(1, max(1, T // 4), T // 2, T, 0.2),
                                    rng_seed=seed, feature_dim=16, edge_attachment=attach)
    g = graphstore.generate(spec)
    cases.append((name, g, prof, cap if cap is not None else default_size_cap(g, 2)))

out = {}
for name, g, prof, cap in cases:
    t0 = time.time()
    cg = propagate(g, prof, cap, 100)
    dt = time.time() - t0
    out[f"{name}/spatial"] = g.spatial_edge_index().astype(np.int64)
    out[f"{name}/temporal"] = g.temporal_link_index().astype(np.int64)
    out[f"{name}/tw"] = _temporal_link_weights(g, prof).astype(np.int64)
    out[f"{name}/meta"] = np.array([g.n_instances, edge_traffic(prof, "spatial"), cap, 100], np.int64)
    out[f"{name}/chunk_of"] = chunk_of(g, cg)
    print(f"{name}: n={g.n_instances} chunks={len(cg.chunks)} cap={cap} reference propagate {dt:.2f}s")
np.savez_compressed(ROOT / "tests" / "golden" / "propagate.npz", **out)
