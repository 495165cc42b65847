"""Native synthetic dynamic-graph generator.

``generate(spec)`` takes the reference's ``SyntheticSpec`` (or any object with
its fields, graphstore.py:385-420) and returns a ``GeneratedGraph`` built by
the native ``dgc_generate_graph`` (csrc/generate.cpp): the contract of
``dynpart.graphstore.generate`` (graphstore.py:525-579) with its own random
stream -- presence runs, clipped-normal per-snapshot edge counts renormalised by
largest remainder, uniform or preferential distinct-pair sampling. The graph's
index views follow the reference's orders exactly (instances snapshot-major,
entity-ascending; spatial edges by snapshot in sorted-pair order; temporal
links earlier presence first), and ``to_dynamic_graph()`` hands it to the
reference planner unchanged (C5: 10M instances x 128 snapshots in seconds
instead of ~25 minutes of reference Python).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native

_KINDS = {"constant": 0, "uniform": 1, "bimodal": 2, "geometric": 3}


class _LengthDist(C.Structure):
    _fields_ = [("kind", C.c_int32), ("value", C.c_int32), ("low", C.c_int32),
                ("high", C.c_int32), ("long_low", C.c_int32), ("long_high", C.c_int32),
                ("long_fraction", C.c_double), ("mean", C.c_double)]


class _Spec(C.Structure):
    _fields_ = [("total_vertices", C.c_int64), ("total_edges", C.c_int64), ("T", C.c_int32),
                ("edges_per_snapshot_mean", C.c_double),
                ("edges_per_snapshot_stddev", C.c_double), ("length", _LengthDist),
                ("rng_seed", C.c_uint64), ("preferential", C.c_int32)]


@dataclass
class GeneratedGraph:
    """A generated dynamic graph: presences [N, 2] (entity, t) and edges
    [E, 3] (t, u, v) as the reference would hold them, plus its index views."""
    T: int
    feature_dim: int
    presences: np.ndarray
    edges: np.ndarray
    n_entities: int

    @property
    def n_instances(self) -> int:
        return int(self.presences.shape[0])

    @property
    def n_spatial_edges(self) -> int:
        return int(self.edges.shape[0])

    def instance_order(self) -> np.ndarray:
        """Presence rows in the global instance order (snapshot-major,
        entity-ascending; graphstore.py:110-118)."""
        return np.lexsort((self.presences[:, 0], self.presences[:, 1]))

    def instances(self) -> np.ndarray:
        """[N, 2] (entity, t) in global instance order."""
        return self.presences[self.instance_order()]

    def _index(self):
        inst = self.instances()
        key = inst[:, 1].astype(np.int64) * (self.n_entities + 1) + inst[:, 0]
        return key  # ascending by construction

    def spatial_edge_index(self) -> np.ndarray:
        """(E, 2) instance indices, snapshot order, sorted pairs (graphstore.py:209-216)."""
        key = self._index()
        e = self.edges.astype(np.int64)
        base = e[:, 0] * (self.n_entities + 1)
        return np.stack([np.searchsorted(key, base + e[:, 1]),
                         np.searchsorted(key, base + e[:, 2])], 1)

    def temporal_link_index(self) -> np.ndarray:
        """(L, 2) instance indices of consecutive presences of each entity, earlier
        first; entities ascending, then time (graphstore.py:172-179, 218-221)."""
        inst = self.instances()
        by_ent = np.lexsort((inst[:, 1], inst[:, 0]))  # entity, then t
        same = inst[by_ent[1:], 0] == inst[by_ent[:-1], 0]
        return np.stack([by_ent[:-1][same], by_ent[1:][same]], 1).astype(np.int64)

    def to_dynamic_graph(self):
        """The reference DynamicGraph of the same presences and edges (validates
        every invariant; needs the reference importable)."""
        from dynpart.graphstore import DynamicGraph
        return DynamicGraph(self.T, self.feature_dim, map(tuple, self.presences.tolist()),
                            map(tuple, self.edges.tolist()))


def generate(spec, n_threads: int = 0) -> GeneratedGraph:
    """dynpart.graphstore.generate's contract on the native generator. Raises
    ValueError for an invalid spec or an infeasible snapshot quota (the
    reference's ValueError / InfeasibleSpecError)."""
    d = spec.presence_length_distribution
    ld = _LengthDist(_KINDS[d.kind], int(getattr(d, "value", 1) or 1), int(getattr(d, "low", 1) or 1),
                     int(getattr(d, "high", 1) or 1), int(getattr(d, "long_low", 1) or 1),
                     int(getattr(d, "long_high", 1) or 1), float(getattr(d, "long_fraction", 0.0) or 0.0),
                     float(getattr(d, "mean", 1.0) or 1.0))
    if spec.edge_attachment not in ("uniform", "preferential"):
        raise ValueError("edge_attachment must be 'uniform' or 'preferential'")
    sp = _Spec(int(spec.total_vertices), int(spec.total_edges), int(spec.T),
               float(spec.edges_per_snapshot_mean), float(spec.edges_per_snapshot_stddev), ld,
               int(spec.rng_seed) & (2 ** 64 - 1), int(spec.edge_attachment == "preferential"))
    if sp.total_vertices < 1:
        raise ValueError("total_vertices must be >= 1")
    if sp.total_edges < 0:
        raise ValueError("total_edges must be >= 0")
    pres = np.empty((max(sp.total_vertices, 0), 2), np.int32)
    edges = np.empty((max(sp.total_edges, 0), 3), np.int32)
    n_ent = C.c_int64()
    lib = _native.lib()
    rc = lib.dgc_generate_graph(C.byref(sp), pres.ctypes.data_as(C.c_void_p),
                                edges.ctypes.data_as(C.c_void_p), C.byref(n_ent), int(n_threads))
    if rc == -1:
        raise ValueError(lib.dgc_last_error().decode())
    _native.check(rc, "dgc_generate_graph")
    return GeneratedGraph(int(spec.T), int(getattr(spec, "feature_dim", 2)), pres, edges,
                          int(n_ent.value))
