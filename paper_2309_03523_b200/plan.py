"""The reference plan, consumed unchanged, as flat arrays.

Three ways in (all yield identical ``PlanArrays``, tests/test_layout.py):
  * ``from_dynpart(g, plan)``: a live ``dynpart.DynamicGraph`` + ``dynpart.Plan``
    from ``build_plan`` (sim.py:167-253), duck-typed -- the drop-in path;
  * ``from_reference_artifacts(dir)``: the reference CLI's stage artifacts
    graph.dg / chunks.json / assignment.json / fusion.json (cli.py:27-33,
    graphstore.py:239-301, partition.py:416-454, assign.py:36-50,
    fusion.py:86-105);
  * ``load_plan_npz(path)``: the compact freeze written by
    tools/make_artifacts.py (used on the GPU box, where the reference is absent).
Global instance order is snapshot-major, entity-ascending
(graphstore.py:68-70,111-122) in every case.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np


class PlanGraphMismatch(ValueError):
    """The plan was built for a different graph (sim.py:108-109)."""


@dataclass
class PlanArrays:
    T: int
    feature_dim: int
    inst_entity: np.ndarray      # int32 [N]
    inst_t: np.ndarray           # int32 [N]
    spatial_edges: np.ndarray    # int32 [E,2]
    temporal_links: np.ndarray   # int32 [L,2]
    structure_device: np.ndarray # int32 [N]
    chunk_of: np.ndarray         # int32 [N]
    n_devices: int
    group_device: np.ndarray | None = None  # int32 [G]
    group_ptr: np.ndarray | None = None     # int64 [G+1]
    group_chunks: np.ndarray | None = None  # int32
    profile: dict = field(default_factory=dict)
    meta: dict = field(default_factory=dict)

    @property
    def n_instances(self) -> int:
        return int(len(self.inst_entity))

    @property
    def n_spatial_edges(self) -> int:
        return int(len(self.spatial_edges))

    @property
    def fused(self) -> bool:
        return self.group_device is not None and len(self.group_device) > 0

    def validate(self) -> None:
        n = self.n_instances
        if len(self.structure_device) != n or len(self.chunk_of) != n:
            raise PlanGraphMismatch(
                f"plan covers {len(self.structure_device)} instances, graph has {n}")
        if n and (self.structure_device.min() < 0 or self.structure_device.max() >= self.n_devices):
            raise PlanGraphMismatch("structure_device out of range for n_devices")
        for arr in (self.spatial_edges, self.temporal_links):
            if len(arr) and (arr.min() < 0 or arr.max() >= n):
                raise PlanGraphMismatch("edge index outside the instance range")


def _i32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def load_plan_npz(path) -> PlanArrays:
    z = dict(np.load(path))
    meta = json.loads(bytes(z["meta"]).decode())
    if "graph_npz" in meta:  # plans of one graph share a graph file (artifacts/<g>_graph.npz)
        g = np.load(Path(path).parent.parent / meta["graph_npz"])
        for k in ("inst_entity", "inst_t", "spatial_edges", "temporal_links"):
            z[k] = g[k]
    fused = bool(meta.get("fused")) and len(z["group_device"]) > 0
    pa = PlanArrays(
        T=int(meta["T"]), feature_dim=int(meta["feature_dim"]),
        inst_entity=_i32(z["inst_entity"]), inst_t=_i32(z["inst_t"]),
        spatial_edges=_i32(z["spatial_edges"]).reshape(-1, 2),
        temporal_links=_i32(z["temporal_links"]).reshape(-1, 2),
        structure_device=_i32(z["structure_device"]), chunk_of=_i32(z["chunk_of"]),
        n_devices=int(meta["n_devices"]),
        group_device=_i32(z["group_device"]) if fused else None,
        group_ptr=np.ascontiguousarray(z["group_ptr"].astype(np.int64)) if fused else None,
        group_chunks=_i32(z["group_chunks"]) if fused else None,
        profile=meta.get("profile", {}), meta=meta)
    pa.validate()
    return pa


def _graph_arrays_from_text(text: str):
    """Parse the reference's .dg format (graphstore.py:239-277) into arrays in
    the reference's global instance order."""
    T = fd = None
    pres, edges = [], []
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        p = line.split()
        if p[0] == "dg":
            T, fd = int(p[1]), int(p[2])
        elif p[0] == "v":
            pres.append((int(p[2]), int(p[1])))  # (t, entity)
        elif p[0] == "e":
            t, u, v = int(p[1]), int(p[2]), int(p[3])
            edges.append((t, min(u, v), max(u, v)))
    if T is None:
        raise ValueError("missing 'dg <T> <feature_dim>' header")
    pres = np.asarray(sorted(set(pres)), dtype=np.int64).reshape(-1, 2)
    inst_t, inst_e = pres[:, 0], pres[:, 1]
    key = inst_t * (int(inst_e.max()) + 1 if len(inst_e) else 1) + inst_e
    stride = int(inst_e.max()) + 1 if len(inst_e) else 1
    edges = np.asarray(sorted(set(edges)), dtype=np.int64).reshape(-1, 3)
    su = np.searchsorted(key, edges[:, 0] * stride + edges[:, 1])
    sv = np.searchsorted(key, edges[:, 0] * stride + edges[:, 2])
    order = np.lexsort((inst_t, inst_e))
    same = inst_e[order][1:] == inst_e[order][:-1]
    tl = np.stack([order[:-1][same], order[1:][same]], axis=1)
    return T, fd, inst_e, inst_t, np.stack([su, sv], axis=1), tl


def from_reference_artifacts(directory) -> PlanArrays:
    d = Path(directory)
    T, fd, inst_e, inst_t, se, tl = _graph_arrays_from_text((d / "graph.dg").read_text())
    stride = int(inst_e.max()) + 1
    key = inst_t * stride + inst_e
    chunks = json.loads((d / "chunks.json").read_text())
    chunk_of = np.full(len(inst_e), -1, np.int64)
    for c in chunks["chunks"]:
        m = np.asarray(c["members"], dtype=np.int64).reshape(-1, 2)
        chunk_of[np.searchsorted(key, m[:, 1] * stride + m[:, 0])] = c["id"]
    asg = json.loads((d / "assignment.json").read_text())
    dev_of_chunk = {c: dv for dv, q in enumerate(asg["queues"]) for c in q}
    sdev = np.asarray([dev_of_chunk[int(c)] for c in chunk_of], dtype=np.int32)
    gd = gp = gc = None
    fpath = d / "fusion.json"
    if fpath.exists():
        fus = json.loads(fpath.read_text())
        gdev, gptr, gch = [], [0], []
        for dv, glist in sorted(((int(k), v) for k, v in fus["devices"].items())):
            for grp in glist:
                gdev.append(dv)
                gch.extend(grp["chunks"])
                gptr.append(len(gch))
        gd, gp, gc = _i32(gdev), np.asarray(gptr, np.int64), _i32(gch)
    pa = PlanArrays(T=T, feature_dim=fd, inst_entity=_i32(inst_e), inst_t=_i32(inst_t),
                    spatial_edges=_i32(se), temporal_links=_i32(tl), structure_device=sdev,
                    chunk_of=_i32(chunk_of), n_devices=len(asg["queues"]), group_device=gd,
                    group_ptr=gp, group_chunks=gc, profile=chunks.get("profile", {}))
    pa.validate()
    return pa


def from_dynpart(g, plan) -> PlanArrays:
    """Duck-typed adapter for a live reference DynamicGraph + Plan.

    The B200 step runs the time encoder on the structure device (the chunk
    plans of the reference, ``Plan.time_device is None``, sim.py:119-121); a
    pss-ts plan, whose time phase moves instances to other devices
    (sim.py:243-252), is rejected instead of being silently re-homed."""
    tdev = getattr(plan, "time_device", None)
    if tdev is not None and not np.array_equal(np.asarray(tdev), np.asarray(plan.structure_device)):
        raise ValueError(f"plan method {getattr(plan, 'method', '?')!r} has a separate time-phase "
                         "device map (pss-ts); the B200 step runs the time encoder on the "
                         "structure device")
    inst = np.asarray(g.instances, dtype=np.int64).reshape(-1, 2)
    chunk_of = np.empty(g.n_instances, np.int64)
    for c in plan.chunk_graph.chunks:
        for v in c.members:
            chunk_of[g.index_of(v)] = c.id
    gd = gp = gc = None
    if plan.fusion is not None:
        gdev, gptr, gch = [], [0], []
        for dv, glist in sorted(plan.fusion.groups_by_device.items()):
            for grp in glist:
                gdev.append(dv)
                gch.extend(grp.chunk_ids)
                gptr.append(len(gch))
        gd, gp, gc = _i32(gdev), np.asarray(gptr, np.int64), _i32(gch)
    prof = plan.messages.profile.to_dict() if hasattr(plan.messages, "profile") else {}
    pa = PlanArrays(T=g.T, feature_dim=g.feature_dim, inst_entity=_i32(inst[:, 0]),
                    inst_t=_i32(inst[:, 1]), spatial_edges=_i32(g.spatial_edge_index()),
                    temporal_links=_i32(g.temporal_link_index()),
                    structure_device=_i32(plan.structure_device), chunk_of=_i32(chunk_of),
                    n_devices=int(plan.n_devices), group_device=gd, group_ptr=gp,
                    group_chunks=gc, profile=prof,
                    meta={"method": str(getattr(plan, "method", "pgc"))})
    pa.validate()
    return pa


def single_device(pa: PlanArrays) -> PlanArrays:
    """The same graph with every instance on device 0 (unpartitioned run)."""
    return PlanArrays(pa.T, pa.feature_dim, pa.inst_entity, pa.inst_t, pa.spatial_edges,
                      pa.temporal_links, np.zeros_like(pa.structure_device), pa.chunk_of, 1,
                      None, None, None, pa.profile, dict(pa.meta))


def native_fusion(pa: PlanArrays, queues, memory_budget: int = 1 << 30,
                  bytes_per_vertex: int = 256, bytes_per_edge: int = 64):
    """plan_fusion (fusion.py:206-220) through the native bit-exact port
    (dgc_plan_spatial_fusion). ``queues`` = Assignment.queues (chunk ids per
    device). Returns (group_device, group_ptr, group_chunks, memory, saved)
    in FusionPlan order (devices ascending, groups by representative id)."""
    import ctypes as C

    from . import _native
    prof = pa.profile
    H, s = int(prof.get("embedding_dim", 16)), int(prof.get("bytes_per_scalar", 4))
    if prof.get("temporal_fanout", "previous-only") != "previous-only":
        raise ValueError("native fusion supports the previous-only temporal fanout")
    ts = int(prof.get("blocks", 1)) * int(prof.get("spatial_msgs_per_block", 2)) * H * s
    tt = int(prof.get("blocks", 1)) * int(prof.get("temporal_msgs_per_block", 1)) * H * s
    se = np.ascontiguousarray(pa.spatial_edges, np.int32).reshape(-1)
    tl = np.ascontiguousarray(pa.temporal_links, np.int32).reshape(-1)
    co = np.ascontiguousarray(pa.chunk_of, np.int32)
    n_chunks = int(co.max()) + 1 if len(co) else 0
    lib = _native.lib()
    gdev, gptr, gch, gmem, gsav = [], [0], [], [], []
    for d, q in enumerate(queues):
        qa = np.ascontiguousarray(np.asarray(q, np.int32))
        goc = np.empty(len(qa), np.int32)
        mem = np.empty(max(1, len(qa)), np.int64)
        sav = np.empty(max(1, len(qa)), np.int64)
        ng = C.c_int64()
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        rc = lib.dgc_plan_spatial_fusion(pa.n_instances, p(se), len(pa.spatial_edges), p(tl),
                                         len(pa.temporal_links), p(co), n_chunks, p(qa), len(qa),
                                         ts, tt, memory_budget, bytes_per_vertex, bytes_per_edge,
                                         p(goc), p(mem), p(sav), C.byref(ng))
        if rc == -3:
            raise ValueError(lib.dgc_last_error().decode())
        _native.check(rc, "dgc_plan_spatial_fusion")
        for gi in range(ng.value):
            members = sorted(int(c) for c in qa[goc == gi])
            gdev.append(d)
            gch.extend(members)
            gptr.append(len(gch))
            gmem.append(int(mem[gi]))
            gsav.append(int(sav[gi]))
    return (np.asarray(gdev, np.int32), np.asarray(gptr, np.int64), np.asarray(gch, np.int32),
            np.asarray(gmem, np.int64), np.asarray(gsav, np.int64))
