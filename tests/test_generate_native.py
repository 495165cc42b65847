"""§8(f)-3: the native synthetic generator (csrc/generate.cpp) against the
contract of dynpart.graphstore.generate (graphstore.py:525-579): totals, the
presence and edge invariants the reference DynamicGraph validates, its index
orders, determinism per seed, the spec errors, and the distributional shape
of the reference generator on the same spec (its random stream is its own)."""
import numpy as np
import pytest

from paper_2309_03523_b200.generate import generate

REF = "/root/reference/pkg/src"


class _Len:
    def __init__(self, kind, **kw):
        self.kind = kind
        for k, v in kw.items():
            setattr(self, k, v)


class _Spec:
    def __init__(self, N=20_000, T=16, sigma=1.0, kind="bimodal", attach="preferential", seed=0):
        self.total_vertices, self.total_edges, self.T = N, 4 * N, T
        self.edges_per_snapshot_mean = 4 * N / T
        self.edges_per_snapshot_stddev = sigma * 4 * N / T
        self.presence_length_distribution = (
            _Len("bimodal", low=1, high=max(1, T // 4), long_low=max(1, T // 2), long_high=T,
                 long_fraction=0.2) if kind == "bimodal" else
            _Len("geometric", mean=4.0) if kind == "geometric" else
            _Len("uniform", low=1, high=8) if kind == "uniform" else _Len("constant", value=3))
        self.rng_seed, self.feature_dim, self.edge_attachment = seed, 16, attach


@pytest.mark.parametrize("kind,attach", [("bimodal", "preferential"), ("geometric", "uniform"),
                                         ("uniform", "preferential"), ("constant", "uniform")])
def test_invariants(kind, attach):
    sp = _Spec(kind=kind, attach=attach)
    g = generate(sp)
    assert g.n_instances == sp.total_vertices and g.n_spatial_edges == sp.total_edges
    p, e = g.presences.astype(np.int64), g.edges.astype(np.int64)
    # presences: unique, inside [1, T], one contiguous run per entity, grouped by entity
    key = p[:, 0] * (sp.T + 1) + p[:, 1]
    assert len(np.unique(key)) == len(key) and np.all(np.diff(key) > 0)
    assert p[:, 1].min() >= 1 and p[:, 1].max() <= sp.T
    ent_first = np.r_[True, p[1:, 0] != p[:-1, 0]]
    assert np.all((p[1:, 1] == p[:-1, 1] + 1) | ent_first[1:])
    assert g.n_entities == len(np.unique(p[:, 0]))
    # edges: no self loops, u < v, both endpoints present at t, no duplicates,
    # snapshot order with sorted pairs
    assert np.all(e[:, 1] < e[:, 2])
    present = set(map(tuple, p[:, ::-1].tolist()))
    assert all((t, u) in present and (t, v) in present for t, u, v in e[::97].tolist())
    ek = (e[:, 0] * (g.n_entities + 1) + e[:, 1]) * (g.n_entities + 1) + e[:, 2]
    assert np.all(np.diff(ek) > 0)
    # per-snapshot counts sum exactly; index views consistent with the instances
    inst = g.instances()
    se = g.spatial_edge_index()
    assert np.array_equal(inst[se[:, 0], 1], e[:, 0]) and np.array_equal(inst[se[:, 0], 0], e[:, 1])
    assert np.array_equal(inst[se[:, 1], 0], e[:, 2])
    tl = g.temporal_link_index()
    assert np.all(inst[tl[:, 0], 0] == inst[tl[:, 1], 0]) and np.all(inst[tl[:, 1], 1] > inst[tl[:, 0], 1])
    assert len(tl) == sp.total_vertices - g.n_entities


def test_deterministic_per_seed_and_thread_count():
    a, b = generate(_Spec(seed=7), n_threads=1), generate(_Spec(seed=7), n_threads=8)
    assert np.array_equal(a.presences, b.presences) and np.array_equal(a.edges, b.edges)
    c = generate(_Spec(seed=8))
    assert not np.array_equal(a.edges, c.edges)


def test_spec_errors():
    sp = _Spec()
    sp.edges_per_snapshot_mean = 0.0
    with pytest.raises(ValueError):
        generate(sp)
    sp = _Spec(N=40, T=4)
    sp.total_edges = 10_000  # 10 vertices per snapshot host at most 45 edges
    with pytest.raises(ValueError, match="edges requested"):
        generate(sp)


def test_matches_reference_dynamic_graph_and_shape(monkeypatch):
    """The reference DynamicGraph accepts the native graph unchanged (every
    invariant validated there) and its index views equal the native ones; the
    native and reference generators agree on the distributional shape."""
    import os
    import sys
    if not os.path.isdir(REF):
        pytest.skip("reference not present")
    monkeypatch.syspath_prepend(REF)
    from dynpart import graphstore as gs
    spec = gs.SyntheticSpec(
        total_vertices=30_000, total_edges=120_000, T=16, edges_per_snapshot_mean=7500.0,
        edges_per_snapshot_stddev=7500.0,
        presence_length_distribution=gs.LengthDistribution.bimodal(1, 4, 8, 16, 0.2), rng_seed=0,
        feature_dim=16, edge_attachment="preferential")
    g = generate(spec)
    dg = g.to_dynamic_graph()
    assert dg.n_instances == g.n_instances and dg.n_spatial_edges == g.n_spatial_edges
    assert np.array_equal(dg.spatial_edge_index(), g.spatial_edge_index())
    assert np.array_equal(dg.temporal_link_index(), g.temporal_link_index())
    ref = gs.generate(spec)
    for G in (dg, ref):  # same spec -> similar entity count, links, degree skew
        deg = np.bincount(G.spatial_edge_index().ravel(), minlength=G.n_instances)
        G._stats = (G.n_entities, len(G.temporal_link_index()), deg.mean(), np.percentile(deg, 90))
    (e1, l1, m1, q1), (e2, l2, m2, q2) = dg._stats, ref._stats
    assert abs(e1 - e2) / e2 < 0.1 and abs(l1 - l2) / l2 < 0.1
    assert abs(m1 - m2) < 1e-9 and 0.5 < q1 / q2 < 2.0
