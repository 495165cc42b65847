"""ctypes binding of the C ABI in include/dgc_b200.h (libdgc_b200.so).

The library is built in-tree (``make`` / ``__graft_entry__.build()``). There is
no fallback: if it is missing, importing any GPU op raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("DGC_LIB_PATH") or
                Path(__file__).resolve().parent / "lib" / "libdgc_b200.so")

_i32, _i64, _f32, _p = C.c_int32, C.c_int64, C.c_float, C.c_void_p


class DgcError(RuntimeError):
    """A native DGC entry point failed (message from dgc_last_error)."""


class PlanView(C.Structure):
    _fields_ = [
        ("n_instances", _i64), ("inst_entity", _p), ("inst_t", _p),
        ("n_spatial_edges", _i64), ("spatial_edges", _p),
        ("n_temporal_links", _i64), ("temporal_links", _p),
        ("structure_device", _p), ("chunk_of", _p), ("n_devices", _i32),
        ("n_groups", _i64), ("group_device", _p), ("group_ptr", _p), ("group_chunks", _p),
        ("segment_rows", _i32),
    ]


_SIGS = {
    "dgc_version": (_i32, []),
    "dgc_to_f16": (_i32, [_p, _p, _i64, _p]),
    "dgc_round_f16": (_i32, [_p, _p, _i64, _p]),
    "dgc_unpack_f16": (_i32, [_p, _p, _i64, _p]),
    "dgc_gemm_f16": (_i32, [_p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _i32, _i32, _f32, _p, _p,
                            _i32, _i32, _p, _p, _p, _i64, _f32, _p, _i64, _p]),
    "dgc_gemm_f16_stacked_a": (_i32, [_p, _i64, _p, _i64, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64,
                                      _i32, _i32, _f32, _i32, _p, _p]),
    "dgc_generate_graph": (_i32, [_p, _p, _p, _p, _i32]),
    "dgc_last_error": (C.c_char_p, []),
    "dgc_layout_build": (_i32, [C.POINTER(PlanView), _i32, C.POINTER(_p)]),
    "dgc_layout_field": (_i64, [_p, _i32, C.POINTER(C.POINTER(_i64))]),
    "dgc_layout_free": (None, [_p]),
    "dgc_plan_spatial_fusion": (_i32, [_i64, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _i64,
                                       _i64, _i64, _i64, _p, _p, _p, _p]),
    "dgc_propagate_labels": (_i32, [_i64, _i64, _p, _i64, _p, _i64, _p, _i64, _i32, _p, _p, _p]),
    "dgc_lstm_fwd_tc_f16x": (_i32, [_p, _i64, _p, _p, _p, _p, _p, _p, _p, _i64, _i32, _i64, _p, _p,
                                    _p, _p, _i32, _p]),
    "dgc_rnn_fwd_tc_fused_available": (_i32, [_i32, _i32]),
    "dgc_pack_sequences": (_i32, [_p, _i64, _i32, _i64, _p, _p, _p, _p, _p]),
    "dgc_spmm_csr": (_i32, [_p, _p, _p, _p, _p, _p, _i64, _i32, _i32, _p]),
    "dgc_gemm_tf32": (_i32, [_p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _i32, _i32, _i32,
                              _p, _p, _i32, _i32, _p, _p, _p]),
    "dgc_gemm_max_ctas": (_i32, [_i32]),
    "dgc_gemm_splits": (_i32, [_i64, _i32, _i32]),
    "dgc_gemm_tf32_stacked_a": (_i32, [_p, _i64, _p, _i64, _i64, _p, _i64, _p, _i64, _i64, _i64,
                                       _i64, _i32, _i32, _i32, _i32, _p, _p]),
    "dgc_gemm_tf32_segmented": (_i32, [_p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _i32, _i32,
                                        _i32, _p, _p, _p, _i32, _p, _i32, _p, _i32, _p, _p, _i32,
                                        _p]),
    "dgc_evolve_fwd": (_i32, [_i32, _i32, _i32] + [_p] * 14 + [_i32, _p]),
    "dgc_evolve_bwd": (_i32, [_i32, _i32, _i32] + [_p] * 16 + [_i32, _p]),
    "dgc_rnn_save_floats": (_i32, [_i32, _i32]),
    "dgc_rnn_fwd": (_i32, [_i32, _p, _p, _p, _p, _p, _p, _i64, _i32, _i32, _i64, _p, _p, _p, _p]),
    "dgc_rnn_fwd_tc": (_i32, [_i32, _p, _p, _p, _p, _p, _p, _i64, _i32, _i32, _i64, _p, _p, _p, _p]),
    "dgc_rnn_bwd": (_i32, [_i32, _p, _p, _p, _i64, _i32, _i32, _p, _p, _p, _p, _p]),
    "dgc_rnn_bwd_tc": (_i32, [_i32, _p, _p, _p, _i64, _i32, _i32, _p, _p, _p, _p, _p, _p]),
    "dgc_rnn_tc_tiles": (_i64, [_i64, _i32]),
    "dgc_rnn_tc_save_floats": (_i32, [_i32]),
    "dgc_rnn_bwd_partial_rows": (_i64, [_i64, _i32]),
    "dgc_transpose": (_i32, [_p, _i64, _i64, _p, _p]),
    "dgc_stale_distance": (_i32, [_p, _p, _p, _p, _i64, _i32, _p, _p, _p]),
    "dgc_stale_select": (_i32, [_p, _p, _p, _f32, _p, _p, _p, _i64, _i32, _p]),
    "dgc_compact_sent": (_i32, [_p, _i64, _p, _p, _p, _p]),
    "dgc_spmm_csr_rows": (_i32, [_p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i32, _i32, _p]),
    "dgc_spmm_csr_h": (_i32, [_p, _p, _p, _p, _p, _p, _p, _f32, _i64, _i32, _i32, _p, _p]),
    "dgc_spmm_csr_x": (_i32, [_p, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i32, _i32, _p, _f32, _p]),
    "dgc_stale_select2": (_i32, [_p, _p, _p, C.c_double, _p, C.c_double, _p, _p, _p, _i64, _i32,
                                 _p, _p, _p]),
    "dgc_exchange_rank": (_i32, [_p, _i64, _p, _i32, _p, _p, _p, _p]),
    "dgc_exchange_pack": (_i32, [_p, _i32, _p, _p, _p, _p, _i64, _p, _p]),
    "dgc_exchange_unpack": (_i32, [_p, _i32, _p, _i32, _p, _p, _i64, _p, _p]),
    "dgc_exchange_pack_back": (_i32, [_p, _i32, _p, _i32, _p, _p, _i64, _p, _p, _p]),
    "dgc_exchange_add_back": (_i32, [_p, _i32, _p, _p, _p, _p, _i64, _p, _p]),
    "dgc_gather_rows": (_i32, [_p, _p, _p, _i64, _i32, _p, _p]),
    "dgc_scatter_rows": (_i32, [_p, _p, _p, _i64, _i32, _p, _i32, _p]),
    "dgc_softmax_xent": (_i32, [_p, _p, _i64, _i32, _f32, _i32, _p, _p, _p, _p]),
    "dgc_softmax_xent_f16": (_i32, [_p, _p, _i64, _i32, _f32, _p, _p, _p, _p, _f32, _p]),
    "dgc_readout_f16": (_i32, [_p, _p, _p, _p, _i64, _i32, _i32, _f32, _f32, _p, _p, _p, _p, _p]),
    "dgc_readout_f16_grid": (_i32, [_i64]),
    "dgc_zero_async": (_i32, [_p, _i64, _p]),
    "dgc_readout_f16_evolve": (_i32, [_p, _p, _p, _p, _i64, _i32, _i32, _f32, _f32, _p, _p, _p, _p, _p, _p]),
    "dgc_reduce_rows_batched": (_i32, [_i32, _p, _p, _p, _p, _p]),
    "dgc_reduce_rows": (_i32, [_p, _i64, _i32, _p, _i32, _p]),
    "dgc_unpack_tf32x24": (_i32, [_p, _p, _i64, _p]),
    "dgc_round_tf32": (_i32, [_p, _p, _i64, _p]),
    "dgc_colsum": (_i32, [_p, _i64, _i32, _i64, _p, _i32, _p, _p]),
    "dgc_relu_bwd": (_i32, [_p, _p, _p, _i64, _p]),
    "dgc_sgd": (_i32, [_p, _p, _p, _i64, _f32, _f32, _p]),
    "dgc_adam": (_i32, [_p, _p, _p, _p, _i64, _f32, _f32, _f32, _f32, _i32, _p]),
    "dgc_adam_dev": (_i32, [_p, _p, _p, _p, _i64, _f32, _f32, _f32, _f32, _p, _p]),
    "dgc_adam_dev_mirror": (_i32, [_p, _p, _p, _p, _i64, _f32, _f32, _f32, _f32, _p, _p, _p, _p]),
    "dgc_epoch_finish": (_i32, [_p, _i64, _p, _p, _p]),
}

_lib = None


def lib():
    """Load libdgc_b200.so once; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DgcError(
                f"native library missing: {LIB_PATH} (run `make` or __graft_entry__.build()); "
                "there is no CPU fallback")
        _lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
        for name, (res, args) in _SIGS.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().dgc_last_error().decode(errors="replace")
        raise DgcError(f"{what or 'dgc'} failed ({rc}): {msg}")
