"""Chunk generation (PGC) through the native, bit-exact port of the
reference's weighted label propagation (dgc_propagate_labels,
csrc/propagate.cpp; partition.py:200-270).

``propagate(g, profile, size_cap, max_rounds)`` keeps the reference's
signature and returns its ChunkGraph (built by the reference's own
_build_chunk_graph from the native labels), so ``native_planner()`` can swap
it into ``dynpart.sim.build_plan`` unchanged: same chunks, same ids, in
seconds instead of minutes at 1M instances. The numpy
entry point ``propagate_labels`` needs no reference import.
"""
from __future__ import annotations

import contextlib
import ctypes as C

import numpy as np

from . import _native


def propagate_labels(n_instances: int, spatial_edges, temporal_links, spatial_weight: int,
                     temporal_weights, size_cap: int, max_rounds: int = 100):
    """Final PGC label per instance (int64 [n]) plus (rounds run, colour
    classes). Inputs as DynamicGraph.spatial_edge_index() /
    temporal_link_index() (reference order), edge_traffic(profile, "spatial")
    and _temporal_link_weights(g, profile)."""
    se = np.ascontiguousarray(np.asarray(spatial_edges, np.int64).reshape(-1, 2))
    tl = np.ascontiguousarray(np.asarray(temporal_links, np.int64).reshape(-1, 2))
    tw = np.ascontiguousarray(np.asarray(temporal_weights, np.int64).reshape(-1))
    if len(tw) != len(tl):
        raise ValueError("temporal_weights must have one weight per temporal link")
    labels = np.empty(int(n_instances), np.int64)
    rounds, colors = C.c_int32(), C.c_int32()
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    rc = _native.lib().dgc_propagate_labels(int(n_instances), len(se), p(se), len(tl), p(tl),
                                            int(spatial_weight), p(tw), int(size_cap),
                                            int(max_rounds), p(labels), C.byref(rounds),
                                            C.byref(colors))
    if rc == -1:  # DGC_ERR_ARG: the reference raises ValueError for the same inputs
        raise ValueError(_native.lib().dgc_last_error().decode())
    _native.check(rc, "dgc_propagate_labels")
    return labels, rounds.value, colors.value


def chunk_ids(labels: np.ndarray) -> np.ndarray:
    """Chunk id per instance = rank of its label (partition.py:298)."""
    return np.unique(labels, return_inverse=True)[1].astype(np.int64)


def propagate(g, profile, size_cap: int, max_rounds: int = 100):
    """dynpart.partition.propagate (partition.py:200-270) with the label
    computation on the native port; the ChunkGraph is assembled by the
    reference's _build_chunk_graph (needs the reference importable)."""
    from dynpart.costmodel import edge_traffic
    from dynpart.partition import _build_chunk_graph, _temporal_link_weights
    if size_cap < 1:
        raise ValueError("size_cap must be >= 1")
    if max_rounds < 1:
        raise ValueError("max_rounds must be >= 1")
    labels, _, _ = propagate_labels(g.n_instances, g.spatial_edge_index(), g.temporal_link_index(),
                                    edge_traffic(profile, "spatial"),
                                    _temporal_link_weights(g, profile), size_cap, max_rounds)
    return _build_chunk_graph(g, profile, labels)


@contextlib.contextmanager
def native_planner():
    """Run dynpart.sim.build_plan with the native propagate (same plan)."""
    import dynpart.partition as dp
    import dynpart.sim as ds
    old = (dp.propagate, ds.propagate)
    dp.propagate = ds.propagate = propagate
    try:
        yield
    finally:
        dp.propagate, ds.propagate = old
