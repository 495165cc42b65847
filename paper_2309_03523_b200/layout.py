"""Per-device layout from the native builder (csrc/layout.cpp, C ABI
dgc_layout_build) -- the plan -> device-tensor boundary of SURVEY.md §8(b)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native
from .plan import PlanArrays, PlanGraphMismatch

FIELDS = ["own_gid", "halo_gid", "group_ptr", "row_ptr", "col", "deg", "t_row_ptr", "t_col",
          "key_rows", "send_ptr", "send_pos", "recv_ptr", "recv_slot", "run_ptr", "run_rows",
          "run_pred_gid", "run_carry", "slot_row", "slot_mask", "slot_carry", "tkey_rows",
          "tsend_ptr", "tsend_pos", "trecv_ptr", "trecv_carry", "scalars", "key_ncut", "seg_ptr"]


@dataclass
class DeviceLayout:
    device: int
    n_devices: int
    arrays: dict

    def __getattr__(self, name):
        a = self.__dict__.get("arrays")
        if a is not None and name in a:
            return a[name]
        raise AttributeError(name)

    @property
    def n_own(self):
        return int(self.arrays["scalars"][0])

    @property
    def n_halo(self):
        return int(self.arrays["scalars"][1])

    @property
    def n_rows(self):
        return int(self.arrays["scalars"][2])

    @property
    def row_len(self):
        return int(self.arrays["scalars"][3])

    @property
    def padding(self):
        return int(self.arrays["scalars"][4])

    @property
    def naive_padding(self):
        return int(self.arrays["scalars"][5])

    @property
    def n_carry(self):
        return int(self.arrays["scalars"][6])

    @property
    def loaded_rows(self):
        return int(self.arrays["scalars"][7])

    @property
    def nnz(self):
        return int(self.arrays["row_ptr"][-1])

    @property
    def dinv(self):
        return (1.0 / np.sqrt(self.arrays["deg"].astype(np.float64) + 1.0))

    @property
    def real_rows(self):
        """mask of own rows that are instances (False on snapshot padding rows)"""
        return self.arrays["own_gid"] >= 0


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def build_layout(pa: PlanArrays, device: int, segment_rows: int = 0) -> DeviceLayout:
    pa.validate()
    lib = _native.lib()
    keep = dict(e=np.ascontiguousarray(pa.inst_entity, np.int32),
                t=np.ascontiguousarray(pa.inst_t, np.int32),
                se=np.ascontiguousarray(pa.spatial_edges, np.int32).reshape(-1),
                tl=np.ascontiguousarray(pa.temporal_links, np.int32).reshape(-1),
                sd=np.ascontiguousarray(pa.structure_device, np.int32),
                co=np.ascontiguousarray(pa.chunk_of, np.int32))
    pv = _native.PlanView()
    pv.n_instances = pa.n_instances
    pv.inst_entity, pv.inst_t = _ptr(keep["e"]), _ptr(keep["t"])
    pv.n_spatial_edges, pv.spatial_edges = len(pa.spatial_edges), _ptr(keep["se"])
    pv.n_temporal_links, pv.temporal_links = len(pa.temporal_links), _ptr(keep["tl"])
    pv.structure_device, pv.chunk_of = _ptr(keep["sd"]), _ptr(keep["co"])
    pv.n_devices = pa.n_devices
    if pa.fused:
        keep["gd"] = np.ascontiguousarray(pa.group_device, np.int32)
        keep["gp"] = np.ascontiguousarray(pa.group_ptr, np.int64)
        keep["gc"] = np.ascontiguousarray(pa.group_chunks, np.int32)
        pv.n_groups = len(pa.group_device)
        pv.group_device, pv.group_ptr, pv.group_chunks = _ptr(keep["gd"]), _ptr(keep["gp"]), _ptr(keep["gc"])
    else:
        pv.n_groups = 0
    pv.segment_rows = int(segment_rows)
    handle = C.c_void_p()
    rc = lib.dgc_layout_build(C.byref(pv), device, C.byref(handle))
    if rc == -3:
        raise PlanGraphMismatch(lib.dgc_last_error().decode())
    _native.check(rc, "dgc_layout_build")
    try:
        arrays = {}
        for i, name in enumerate(FIELDS):
            ptr = C.POINTER(C.c_int64)()
            n = lib.dgc_layout_field(handle, i, C.byref(ptr))
            arrays[name] = np.ctypeslib.as_array(ptr, shape=(n,)).copy() if n > 0 else np.zeros(0, np.int64)
    finally:
        lib.dgc_layout_free(handle)
    return DeviceLayout(device, pa.n_devices, arrays)


def pack_sequences_native(lengths):
    """fusion.py:278-313 via the native FFD (dgc_pack_sequences).
    Returns (slot_seq [R,L], slot_pos [R,L], mask uint8 [R,L], padding)."""
    lengths = np.ascontiguousarray(np.asarray(lengths, dtype=np.int32))
    n = len(lengths)
    if n == 0:
        z = np.zeros((0, 0), np.int32)
        return z, z, np.zeros((0, 0), np.uint8), 0
    L = int(lengths.max())
    cap = n
    seq = np.empty(cap * L, np.int32)
    pos = np.empty(cap * L, np.int32)
    mask = np.empty(cap * L, np.uint8)
    R = C.c_int64()
    pad = C.c_int64()
    lib = _native.lib()
    _native.check(lib.dgc_pack_sequences(_ptr(lengths), n, L, cap, _ptr(seq), _ptr(pos), _ptr(mask),
                                         C.byref(R), C.byref(pad)), "dgc_pack_sequences")
    r = R.value
    return (seq[:r * L].reshape(r, L), pos[:r * L].reshape(r, L), mask[:r * L].reshape(r, L),
            pad.value)
