"""Thin torch-tensor wrappers over the C ABI (include/dgc_b200.h).

PyTorch is plumbing here: device memory, the current stream and NCCL. Every
function validates dtype/device/contiguity and launches exactly the native
kernel named in its docstring on the current CUDA stream; there is no
fallback path.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native

_NULL = None

# Optional per-launch profiler (bench.py): records CUDA events around every
# native call on the current stream with its algorithmic bytes / flops.
_prof = None
_prof_detail = False


class profile:
    """Context manager collecting (name, start, end, bytes, flops, kernels)."""

    def __init__(self):
        self.records = []

    def __enter__(self):
        global _prof
        _prof = self.records
        return self

    def __exit__(self, *exc):
        global _prof
        _prof = None

    def summary(self):
        torch.cuda.synchronize()
        out = {}
        for name, s, e, nbytes, flops, nk in self.records:
            d = out.setdefault(name, dict(ms=0.0, launches=0, kernels=0, bytes=0.0, flops=0.0))
            d["ms"] += s.elapsed_time(e)
            d["launches"] += 1
            d["kernels"] += nk
            d["bytes"] += nbytes
            d["flops"] += flops
        return out


def _run(name, fn, nbytes=0.0, flops=0.0, kernels=1):
    if _prof is None:
        return fn()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    rc = fn()
    e.record()
    _prof.append((name, s, e, float(nbytes), float(flops), kernels))
    return rc


def _p(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _req(t, dtype, name):
    if t is None:
        return
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


def spmm_csr(row_ptr, col, dinv, Y, bias, out, act: int, nnz=0, n_cols=0, out16=None, work=None,
             scale16=1.0):
    """K1 dgc_spmm_csr: out = act(dinv_i * sum_c dinv_c Y_c + bias).
    Algorithmic bytes: 4W(n_cols + n_rows) + 4(n_rows+1)
    + 4 nnz (+ 4 n_cols for dinv)."""
    _req(row_ptr, torch.int32, "row_ptr"); _req(col, torch.int32, "col")
    _req(Y, torch.float32, "Y"); _req(out, torch.float32, "out")
    n = row_ptr.numel() - 1
    ref = out if out is not None else out16
    W = ref.shape[-1] if ref.dim() > 1 else 1
    nb = (4 * W * n_cols + (4 * W * n if out is not None else 0) + 4 * (n + 1) + 4 * nnz
          + 4 * n_cols + (2 * W * n if out16 is not None else 0))
    _run("spmm_csr", lambda: _native.check(_native.lib().dgc_spmm_csr_x(
        _p(row_ptr), _p(col), _p(dinv), _p(Y), _p(bias), _p(out), _p(out16), None, n, 0, W, act,
        _p(work), float(scale16), _stream()), "dgc_spmm_csr_x"), nb, 2 * nnz * W)
    return out


def spmm_csr_h(row_ptr, col, dinv, Y16, bias, out, act: int, nnz=0, n_cols=0, work=None,
               out16=None, scale16=1.0, name="spmm_csr"):
    """K1 with an fp16 gathered operand (dgc_spmm_csr_h), all rows; fp32 out
    and / or fp16(scale16 * out) in out16."""
    _req(row_ptr, torch.int32, "row_ptr"); _req(col, torch.int32, "col"); _req16(Y16, "Y16")
    _req(out, torch.float32, "out"); _req16(out16, "out16")
    n = row_ptr.numel() - 1
    W = (out if out is not None else out16).shape[-1]
    nb = (2 * W * n_cols + (4 * W * n if out is not None else 0) + (2 * W * n if out16 is not None else 0)
          + 4 * (n + 1) + 4 * nnz + 4 * n_cols)
    _run(name, lambda: _native.check(_native.lib().dgc_spmm_csr_h(
        _p(row_ptr), _p(col), _p(dinv), _p(Y16), _p(bias), _p(out), _p(out16), float(scale16), n, W,
        act, _p(work), _stream()), "dgc_spmm_csr_h"), nb, 2 * nnz * W)
    return out


def spmm_csr_rows(row_ptr, col, dinv, Y, bias, out, act: int, rows=None, n_rows=0, row_begin=0,
                  nnz=0, n_cols=0, name="spmm_csr", out16=None, work=None, scale16=1.0):
    """K1 over a row subset (dgc_spmm_csr_rows): the rows of the int32 list
    ``rows``, or the range [row_begin, row_begin + n_rows). nnz / n_cols: the
    subset's nonzeros and distinct gathered columns (algorithmic bytes)."""
    _req(row_ptr, torch.int32, "row_ptr"); _req(col, torch.int32, "col")
    _req(Y, torch.float32, "Y"); _req(out, torch.float32, "out"); _req(rows, torch.int32, "rows")
    n = rows.numel() if rows is not None else int(n_rows)
    ref = out if out is not None else out16
    W = ref.shape[-1] if ref.dim() > 1 else 1
    nb = 4 * W * (n_cols + n) + 8 * n + 4 * nnz + 4 * n_cols + (2 * W * n if out16 is not None else 0)
    _run(name, lambda: _native.check(_native.lib().dgc_spmm_csr_x(
        _p(row_ptr), _p(col), _p(dinv), _p(Y), _p(bias), _p(out), _p(out16), _p(rows), n,
        int(row_begin), W, act, _p(work), float(scale16), _stream()), "dgc_spmm_csr_x"), nb,
        2 * nnz * W)
    return out


def stale_select_dev(Y, key_rows, dist, dmax, coef, cache, cached, send, width, ncut=None,
                     billed=None, theta=0.0):
    """K5 decision with theta = coef * dmax[0] on the device (dgc_stale_select2);
    dmax None: the host theta. Accumulates the billed cut messages of sent keys."""
    k = key_rows.numel()
    _run("stale_select", lambda: _native.check(_native.lib().dgc_stale_select2(
        _p(Y), _p(key_rows), _p(dist), float(theta), _p(dmax), float(coef), _p(cache),
        _p(cached), _p(send), k, width, _p(ncut), _p(billed), _stream()), "dgc_stale_select2"),
        k * 18)


def exchange_rank(ent_key, ent_ptr, D, send, ent_slot, counts):
    """dgc_exchange_rank: stale compaction of every peer's send list at once."""
    n = ent_key.numel()
    _run("exchange_rank", lambda: _native.check(_native.lib().dgc_exchange_rank(
        _p(ent_key), n, _p(ent_ptr), int(D), _p(send), _p(ent_slot), _p(counts), _stream()),
        "dgc_exchange_rank"), 13 * n)


def exchange_pack(Y, width, key_rows, ent_key, ent_idx, ent_slot, sendbuf, n_sent=None):
    """dgc_exchange_pack: one record per sent entry, all peers in one buffer."""
    n = ent_key.numel()
    rows = n if n_sent is None else n_sent
    _run("exchange_pack", lambda: _native.check(_native.lib().dgc_exchange_pack(
        _p(Y), int(width), _p(key_rows), _p(ent_key), _p(ent_idx), _p(ent_slot), n,
        _p(sendbuf), _stream()), "dgc_exchange_pack"), 12 * n + rows * (8 * width + 16))


def exchange_unpack(recvbuf, width, rcounts, D, rlist, rlist_ptr, n_max, dst):
    _run("exchange_unpack", lambda: _native.check(_native.lib().dgc_exchange_unpack(
        _p(recvbuf), int(width), _p(rcounts), int(D), _p(rlist), _p(rlist_ptr), int(n_max),
        _p(dst), _stream()), "dgc_exchange_unpack"), n_max * (8 * width + 20))


def exchange_pack_back(fwd_recvbuf, width, rcounts, D, rlist, rlist_ptr, n_max, dY, backbuf):
    _run("exchange_pack_back", lambda: _native.check(_native.lib().dgc_exchange_pack_back(
        _p(fwd_recvbuf), int(width), _p(rcounts), int(D), _p(rlist), _p(rlist_ptr), int(n_max),
        _p(dY), _p(backbuf), _stream()), "dgc_exchange_pack_back"), n_max * (8 * width + 20))


def exchange_add_back(backbuf, width, key_rows, kent_ptr, kent, ent_slot, dY):
    n = key_rows.numel()
    _run("exchange_add_back", lambda: _native.check(_native.lib().dgc_exchange_add_back(
        _p(backbuf), int(width), _p(key_rows), _p(kent_ptr), _p(kent), _p(ent_slot), n, _p(dY),
        _stream()), "dgc_exchange_add_back"), n * 12 * width)


def gemm(A, B, C, M, N, K, *, a_mn=False, b_mn=True, lda=None, ldb=None, ldc=None,
         precision=3, bias=None, relu_src=None, accumulate=False, k_splits=1, partial=None,
         colsum_partial=None, act=0):
    """K2 dgc_gemm_tf32 (tcgen05). Defaults: A [M,K] row-major, B [K,N] row-major.
    act: bit 0 ReLU on the output, bit 1 round the output to TF32."""
    for t, nm in ((A, "A"), (B, "B"), (C, "C")):
        _req(t, torch.float32, nm)
    if partial is None and gemm_splits(K, precision, k_splits) > 1:
        raise ValueError(f"gemm: K={K} needs a split-K partial buffer "
                         f"({gemm_splits(K, precision, k_splits)} splits)")
    lda = lda if lda is not None else (M if a_mn else K)
    ldb = ldb if ldb is not None else (N if b_mn else K)
    ldc = ldc if ldc is not None else N
    splits = gemm_splits(K, precision, k_splits)
    nb = 4 * (M * K + K * N + M * N * (1 + int(accumulate) + int(relu_src is not None)))
    gname = "gemm_tf32" if precision == 1 else "gemm_3xtf32"
    if _prof_detail:
        gname += f"[{M}x{N}x{K} a{int(a_mn)}b{int(b_mn)} s{splits}]"
    _run(gname, lambda: _native.check(
        _native.lib().dgc_gemm_tf32(
            _p(A), lda, _p(B), ldb, _p(C), ldc, M, N, K, int(a_mn), int(b_mn), precision,
            _p(bias), _p(relu_src), int(accumulate) | ((int(act) & 3) << 1), k_splits,
            _p(partial), _p(colsum_partial), _stream()),
        "dgc_gemm_tf32"), nb, 2.0 * M * N * K, 1 + int(splits > 1))
    return C


def gemm_stacked_a(A0, A1, B, C, M0, M, N, K, *, a_mn=False, b_mn=True, lda0=None, lda1=None,
                   ldb=None, ldc=None, precision=3, k_splits=1, partial=None):
    """K2 with op(A) = [op(A0); op(A1)] along M (dgc_gemm_tf32_stacked_a): one
    launch for [dWx; dU] = [x; h_in]^T dgx."""
    for t, nm in ((A0, "A0"), (A1, "A1"), (B, "B"), (C, "C")):
        _req(t, torch.float32, nm)
    if partial is None and gemm_splits(K, precision, k_splits) > 1:
        raise ValueError("gemm_stacked_a: split-K needs a partial buffer")
    lda0 = lda0 if lda0 is not None else (M0 if a_mn else K)
    lda1 = lda1 if lda1 is not None else ((M - M0) if a_mn else K)
    ldb = ldb if ldb is not None else (N if b_mn else K)
    ldc = ldc if ldc is not None else N
    splits = gemm_splits(K, precision, k_splits)
    nb = 4 * (M * K + K * N + M * N)
    gname = "gemm_tf32" if precision == 1 else "gemm_3xtf32"
    if _prof_detail:
        gname += f"[{M}x{N}x{K} a{int(a_mn)}b{int(b_mn)} s{splits} stacked]"
    _run(gname, lambda: _native.check(_native.lib().dgc_gemm_tf32_stacked_a(
        _p(A0), lda0, _p(A1), lda1, M0, _p(B), ldb, _p(C), ldc, M, N, K, int(a_mn), int(b_mn),
        precision, k_splits, _p(partial), _stream()), "dgc_gemm_tf32_stacked_a"),
        nb, 2.0 * M * N * K, 1 + int(splits > 1))
    return C


def _req16(t, name):
    if t is not None and (not t.is_cuda or t.dtype != torch.float16):
        raise ValueError(f"{name} must be a CUDA fp16 tensor")


def gemm_max_ctas(n):
    """dgc_gemm_max_ctas: cap the CTAs of the following GEMM launches (0: all
    SMs); returns the previous cap."""
    return int(_native.lib().dgc_gemm_max_ctas(int(n)))


def gemm_f16(A, B, C, M, N, K, *, a_mn=False, b_mn=True, lda=None, ldb=None, ldc=None, alpha=1.0,
             bias=None, relu_src=None, accumulate=False, k_splits=1, partial=None,
             colsum_partial=None, act=0, C16=None, c16_scale=1.0, relu16=None):
    """K2 with fp16 operands (dgc_gemm_f16): C = alpha * op(A) op(B) [+ epilogue
    as gemm()]; alpha undoes a power-of-two operand scale. C16: fp16(c16_scale *
    C) (C may be None: fp16-only output); relu16: fp16 ReLU-mask source."""
    _req16(A, "A"); _req16(B, "B"); _req(C, torch.float32, "C"); _req16(C16, "C16")
    _req16(relu16, "relu16")
    if partial is None and gemm_splits(K, 2, k_splits) > 1:
        raise ValueError(f"gemm_f16: K={K} needs a split-K partial buffer")
    lda = lda if lda is not None else (M if a_mn else K)
    ldb = ldb if ldb is not None else (N if b_mn else K)
    ldc = ldc if ldc is not None else N
    splits = gemm_splits(K, 2, k_splits)
    nb = (2 * (M * K + K * N) + (4 * M * N if C is not None else 0) * (1 + int(accumulate))
          + 4 * M * N * int(relu_src is not None) + 2 * M * N * (int(C16 is not None)
                                                                 + int(relu16 is not None)))
    gname = "gemm_f16" + (f"[{M}x{N}x{K} a{int(a_mn)}b{int(b_mn)} s{splits}]" if _prof_detail else "")
    ldc16 = C16.stride(0) if C16 is not None else 0
    ldr16 = relu16.stride(0) if relu16 is not None else 0
    _run(gname, lambda: _native.check(_native.lib().dgc_gemm_f16(
        _p(A), lda, _p(B), ldb, _p(C), ldc, M, N, K, int(a_mn), int(b_mn), float(alpha), _p(bias),
        _p(relu_src), int(accumulate) | ((int(act) & 3) << 1), k_splits, _p(partial),
        _p(colsum_partial), _p(C16), ldc16, float(c16_scale), _p(relu16), ldr16, _stream()),
        "dgc_gemm_f16"), nb, 2.0 * M * N * K, 1 + int(splits > 1))
    return C


def gemm_f16_stacked_a(A0, A1, B, C, M0, M, N, K, *, a_mn=False, b_mn=True, lda0=None, lda1=None,
                       ldb=None, ldc=None, alpha=1.0, k_splits=1, partial=None):
    """gemm_stacked_a with fp16 operands (dgc_gemm_f16_stacked_a)."""
    _req16(A0, "A0"); _req16(A1, "A1"); _req16(B, "B"); _req(C, torch.float32, "C")
    if partial is None and gemm_splits(K, 2, k_splits) > 1:
        raise ValueError("gemm_f16_stacked_a: split-K needs a partial buffer")
    lda0 = lda0 if lda0 is not None else (M0 if a_mn else K)
    lda1 = lda1 if lda1 is not None else ((M - M0) if a_mn else K)
    ldb = ldb if ldb is not None else (N if b_mn else K)
    ldc = ldc if ldc is not None else N
    splits = gemm_splits(K, 2, k_splits)
    nb = 2 * (M * K + K * N) + 4 * M * N
    gname = "gemm_f16" + (f"[{M}x{N}x{K} a{int(a_mn)}b{int(b_mn)} s{splits} stacked]" if _prof_detail else "")
    _run(gname, lambda: _native.check(_native.lib().dgc_gemm_f16_stacked_a(
        _p(A0), lda0, _p(A1), lda1, M0, _p(B), ldb, _p(C), ldc, M, N, K, int(a_mn), int(b_mn),
        float(alpha), k_splits, _p(partial), _stream()), "dgc_gemm_f16_stacked_a"),
        nb, 2.0 * M * N * K, 1 + int(splits > 1))
    return C


def gemm_segmented(A, B, C, M, N, K, *, a_mn=False, b_mn=True, lda=None, ldb=None, ldc=None,
                   precision=3, bias=None, relu_src=None, seg_of_mtile=None, b_nseg=1,
                   kitems=None, n_kitems=0, item_ptr=None, n_seg=0, partial=None,
                   colsum_partial=None, act=0):
    """K2 for per-snapshot weights (dgc_gemm_tf32_segmented); act as in gemm()."""
    lda = lda if lda is not None else (M if a_mn else K)
    ldb = ldb if ldb is not None else (N if b_mn else K)
    ldc = ldc if ldc is not None else N
    nb = 4 * (M * K + K * N * max(b_nseg, 1) + M * N * max(1, n_seg))
    gname = "gemm_seg_tf32" if precision == 1 else "gemm_seg_3xtf32"
    if _prof_detail:
        gname += f"[{M}x{N}x{K} a{int(a_mn)}b{int(b_mn)} {'K' if kitems is not None else 'M'}]"
    _run(gname, lambda: _native.check(_native.lib().dgc_gemm_tf32_segmented(
        _p(A), lda, _p(B), ldb, _p(C), ldc, M, N, K, int(a_mn), int(b_mn), precision, _p(bias),
        _p(relu_src), _p(seg_of_mtile), int(b_nseg), _p(kitems), int(n_kitems), _p(item_ptr),
        int(n_seg), _p(partial), _p(colsum_partial), int(act), _stream()),
        "dgc_gemm_tf32_segmented"),
        nb, 2.0 * M * N * K, 1 + int(kitems is not None))
    return C


def evolve_fwd(Fl, Hl, T, W0, Sr, Sz, Pc, Qc, Br, Bz, Bc, Wstack, sv, rnd=False):
    """EvolveGCN-O weight evolution forward (dgc_evolve_fwd); sv = (r, z, c, w, rw)."""
    _run("evolve_fwd", lambda: _native.check(_native.lib().dgc_evolve_fwd(
        Fl, Hl, T, _p(W0), _p(Sr), _p(Sz), _p(Pc), _p(Qc), _p(Br), _p(Bz), _p(Bc),
        _p(Wstack), *[_p(x) for x in sv], int(rnd), _stream()), "dgc_evolve_fwd"),
        4 * T * Fl * Hl * 6 + 16 * T * Fl * Fl, 8.0 * T * Fl * Fl * Hl)


def evolve_bwd(Fl, Hl, T, Sr, Sz, Pc, Qc, sv, dW_direct, dW0, da, dB, rnd=False):
    """EvolveGCN-O weight evolution BPTT (dgc_evolve_bwd); da/dB = (r, z, c) triples."""
    _run("evolve_bwd", lambda: _native.check(_native.lib().dgc_evolve_bwd(
        Fl, Hl, T, _p(Sr), _p(Sz), _p(Pc), _p(Qc), *[_p(x) for x in sv[:4]], _p(dW_direct),
        _p(dW0), *[_p(x) for x in da], *[_p(x) for x in dB], int(rnd), _stream()),
        "dgc_evolve_bwd"), 4 * T * Fl * Hl * 8 + 16 * T * Fl * Fl, 8.0 * T * Fl * Fl * Hl)


def gemm_splits(K, precision, k_splits):
    """Split count dgc_gemm_tf32 will use for a K-long contraction."""
    return _native.lib().dgc_gemm_splits(K, precision, k_splits)


def rnn_save_floats(cell: int, H: int) -> int:
    return _native.lib().dgc_rnn_save_floats(cell, H)


def rnn_fwd(cell, gx, U, slot_row, slot_mask, slot_carry, carry, n_rows, row_len, H, ld_out,
            h_out, c_out, save):
    """K3/K4 dgc_rnn_fwd (masked GRU/LSTM over packed runs)."""
    _req(gx, torch.float32, "gx"); _req(slot_row, torch.int32, "slot_row")
    _req(slot_mask, torch.uint8, "slot_mask"); _req(slot_carry, torch.int32, "slot_carry")
    n_inst, G = gx.shape[0], (3 if cell == 0 else 4)
    sf = rnn_save_floats(cell, H)
    nb = 4 * n_inst * (G * H + sf + H * (1 + cell)) + 9 * n_rows * row_len + 4 * G * H * H
    _run("gru_fwd" if cell == 0 else "lstm_fwd", lambda: _native.check(
        _native.lib().dgc_rnn_fwd(cell, _p(gx), _p(U), _p(slot_row), _p(slot_mask),
                                  _p(slot_carry), _p(carry), n_rows, row_len, H, ld_out,
                                  _p(h_out), _p(c_out), _p(save), _stream()), "dgc_rnn_fwd"),
        nb, 2.0 * n_rows * row_len * H * G * H)


def rnn_fwd_tc(cell, gx, Ut, slot_row, slot_mask, slot_carry, carry, n_rows, row_len, H, ld_out,
               h_out, c_out, save):
    """K4 on tcgen05 (dgc_rnn_fwd_tc): TF32 masked LSTM forward, h x U on tensor cores."""
    _req(gx, torch.float32, "gx"); _req(Ut, torch.float32, "Ut")
    n_inst, G = gx.shape[0], 4
    sf = rnn_save_floats(cell, H)
    nb = 4 * n_inst * (G * H + sf + 2 * H) + 9 * n_rows * row_len + 4 * G * H * H
    _run("lstm_fwd_tc", lambda: _native.check(
        _native.lib().dgc_rnn_fwd_tc(cell, _p(gx), _p(Ut), _p(slot_row), _p(slot_mask),
                                     _p(slot_carry), _p(carry), n_rows, row_len, H, ld_out,
                                     _p(h_out), _p(c_out), _p(save), _stream()),
        "dgc_rnn_fwd_tc"), nb, 2.0 * n_rows * row_len * H * G * H)


def rnn_tc_save_floats(H):
    """Save-row width of the tensor-core LSTM (dgc_rnn_tc_save_floats): 3.5 H
    (h_in fp32 + five fp16 fields) for the H = 128 cluster kernels, else 7 H."""
    return _native.lib().dgc_rnn_tc_save_floats(H)


def rnn_fwd_tc_fused_available(F, H):
    return bool(_native.lib().dgc_rnn_fwd_tc_fused_available(F, H))


def lstm_fwd_tc_f16x(x16, Wx, U, bias, slot_row, slot_mask, slot_carry, carry, n_rows, row_len,
                     H, ld_out, h_out, c_out, save, h_out16=None, c_rows=None,
                     h32_run_ends_only=False):
    """K4 on tcgen05 with the input projection fused (dgc_lstm_fwd_tc_f16x): the
    fp16 x rows of each position are TMA-gathered and multiplied by Wx^T in TMEM
    next to h U^T, both weight halves resident in shared memory as fp16; no gx
    round trip through HBM and no weight traffic per position. With
    h32_run_ends_only (needs h_out16) the fp32 h is written only at run ends."""
    if x16.dtype != torch.float16 or not x16.is_cuda:
        raise ValueError("x16 must be a CUDA fp16 tensor")
    _req(Wx, torch.float32, "Wx"); _req(U, torch.float32, "U")
    n_inst, F = h_out.shape[0], Wx.shape[0]
    G = 4
    # reads x (fp16); writes the save row (h_in fp32 + c_in, i, f, g, o fp16: sf
    # floats; tanh(c) is recomputed by the BPTT), h (+ its fp16 copy), and c at
    # the run ends
    sf = rnn_tc_save_floats(H)
    c_rows = n_inst if c_rows is None else c_rows
    if h32_run_ends_only and h_out16 is None:
        raise ValueError("h32_run_ends_only needs h_out16")
    h32_rows = c_rows if h32_run_ends_only else n_inst
    nb = (n_inst * (2 * F + 4 * sf + (2 * H if h_out16 is not None else 0))
          + 4 * h32_rows * H + 4 * c_rows * H + 9 * n_rows * row_len + 4 * G * H * (H + F))
    _run("lstm_fwd_tc", lambda: _native.check(
        _native.lib().dgc_lstm_fwd_tc_f16x(_p(x16), x16.shape[0], _p(Wx), _p(U), _p(bias),
                                           _p(slot_row), _p(slot_mask), _p(slot_carry), _p(carry),
                                           n_rows, row_len, ld_out, _p(h_out), _p(c_out), _p(save),
                                           _p(h_out16), int(bool(h32_run_ends_only)), _stream()),
        "dgc_lstm_fwd_tc_f16x"),
        nb, 2.0 * n_rows * row_len * H * G * (H + F))


def rnn_bwd_tc(cell, U, slot_row, slot_mask, n_rows, row_len, H, save, dh_out, dgx, dc_scratch,
               bias_partial=None):
    """K4 BPTT on tcgen05 (dgc_rnn_bwd_tc): dh = da U^T on tensor cores. An fp16
    dgx (H = 128 cluster kernel, cell bit 24) receives S * dgx, S = 2^(cell bits
    16..22): the operand of the fp16 weight-gradient GEMMs."""
    dh16 = dh_out.dtype == torch.float16
    if dh16:  # S * dh as fp16 (S = the dgx scale): the K-split cluster BPTT only
        _req16(dh_out, "dh_out")
        cell |= 1 << 25
    else:
        _req(dh_out, torch.float32, "dh_out")
    f16 = dgx.dtype == torch.float16
    if f16:
        _req16(dgx, "dgx")
        if not (H == 128 and rnn_tc_save_floats(H) < 7 * H):
            raise ValueError("rnn_bwd_tc: an fp16 dgx needs the H = 128 cluster kernel")
        cell |= 1 << 24
    else:
        _req(dgx, torch.float32, "dgx")
    n_inst, G = dgx.shape[0], 4
    # reads the saved c_in, i, f, g, o (fp16 in the H = 128 cluster kernel, which
    # recomputes tanh(c); fp32 + tanh(c) otherwise) and dh; writes dgx
    saved_bytes = 2 * 5 * H if rnn_tc_save_floats(H) < 7 * H else 4 * 6 * H
    nb = (n_inst * ((2 if f16 else 4) * G * H + saved_bytes + (2 if dh16 else 4) * H)
          + 5 * n_rows * row_len
          + 4 * G * H * H)
    _run("lstm_bwd_tc", lambda: _native.check(
        _native.lib().dgc_rnn_bwd_tc(cell, _p(U), _p(slot_row), _p(slot_mask), n_rows, row_len, H,
                                     _p(save), _p(dh_out), _p(dgx), _p(dc_scratch),
                                     _p(bias_partial), _stream()), "dgc_rnn_bwd_tc"),
        nb, 2.0 * n_rows * row_len * H * G * H)


def rnn_tc_tiles(n_rows, H):
    """Rows of the tensor-core BPTT's bias partials (dgc_rnn_tc_tiles)."""
    return _native.lib().dgc_rnn_tc_tiles(n_rows, H)


def rnn_bwd_partial_rows(n_rows, H):
    return _native.lib().dgc_rnn_bwd_partial_rows(n_rows, H)


def reduce_rows(partial, rows, width, out, accumulate=False):
    """dgc_reduce_rows: out[j] (+)= sum_r partial[r, j] (fixed order)."""
    _run("reduce_rows", lambda: _native.check(_native.lib().dgc_reduce_rows(
        _p(partial), rows, width, _p(out), int(accumulate), _stream()), "dgc_reduce_rows"),
        4 * rows * width, 0, 2)
    return out


def reduce_rows_batched(jobs):
    """dgc_reduce_rows_batched: jobs = [(partial, rows, width, out), ...] (<= 8),
    bitwise the same as reduce_rows per job, in two launches."""
    import ctypes
    n = len(jobs)
    P = (ctypes.c_void_p * n)(*[p.data_ptr() for p, _, _, _ in jobs])
    R = (ctypes.c_int64 * n)(*[int(r) for _, r, _, _ in jobs])
    W = (ctypes.c_int32 * n)(*[int(w) for _, _, w, _ in jobs])
    O = (ctypes.c_void_p * n)(*[o.data_ptr() for _, _, _, o in jobs])
    _run("reduce_rows", lambda: _native.check(_native.lib().dgc_reduce_rows_batched(
        n, ctypes.addressof(P), ctypes.addressof(R), ctypes.addressof(W), ctypes.addressof(O),
        _stream()), "dgc_reduce_rows_batched"),
        sum(4 * r * w for _, r, w, _ in jobs), 0, 2)


def rnn_bwd(cell, Ut, slot_row, slot_mask, n_rows, row_len, H, save, dh_out, dgx,
            bias_partial=None):
    """K3/K4 dgc_rnn_bwd (BPTT over packed runs)."""
    _req(dh_out, torch.float32, "dh_out"); _req(dgx, torch.float32, "dgx")
    n_inst, G = dgx.shape[0], (3 if cell == 0 else 4)
    sf = rnn_save_floats(cell, H)
    nb = 4 * n_inst * (G * H + sf + H) + 5 * n_rows * row_len + 4 * G * H * H
    _run("gru_bwd" if cell == 0 else "lstm_bwd", lambda: _native.check(
        _native.lib().dgc_rnn_bwd(cell, _p(Ut), _p(slot_row), _p(slot_mask), n_rows, row_len, H,
                                  _p(save), _p(dh_out), _p(dgx), _p(bias_partial), _stream()),
        "dgc_rnn_bwd"),
        nb, 2.0 * n_rows * row_len * H * G * H)


def transpose(x, out):
    _run("transpose", lambda: _native.check(_native.lib().dgc_transpose(
        _p(x), x.shape[0], x.shape[1], _p(out), _stream()), "dgc_transpose"), 8 * x.numel())
    return out


def stale_distance(Y, key_rows, cache, cached, width, dist, dmax):
    """K5 dgc_stale_distance."""
    k = key_rows.numel()
    _run("stale_distance", lambda: _native.check(_native.lib().dgc_stale_distance(
        _p(Y), _p(key_rows), _p(cache), _p(cached), k, width, _p(dist), _p(dmax), _stream()),
        "dgc_stale_distance"), k * (8 * width + 9), 3 * k * width, 2)


def stale_select(Y, key_rows, dist, theta, cache, cached, send, width):
    """K5 dgc_stale_select (strict > theta; theta < 0 sends all)."""
    k = key_rows.numel()
    _run("stale_select", lambda: _native.check(_native.lib().dgc_stale_select(
        _p(Y), _p(key_rows), _p(dist), float(theta), _p(cache), _p(cached), _p(send), k, width,
        _stream()), "dgc_stale_select"), k * 10)


def compact_sent(pos, send, out_idx, count):
    """K6 dgc_compact_sent."""
    _run("compact_sent", lambda: _native.check(_native.lib().dgc_compact_sent(
        _p(pos), pos.numel(), _p(send), _p(out_idx), _p(count), _stream()), "dgc_compact_sent"),
        9 * pos.numel())


def gather_rows(Y, rows, idx, n, width, out):
    """K6 dgc_gather_rows: out[i] = Y[rows[idx[i]]]."""
    _run("gather_rows", lambda: _native.check(_native.lib().dgc_gather_rows(
        _p(Y), _p(rows), _p(idx), n, width, _p(out), _stream()), "dgc_gather_rows"),
        n * (8 * width + 8))
    return out


def scatter_rows(src, rows, idx, n, width, dst, add=False):
    """K6 dgc_scatter_rows: dst[rows[idx[i]]] (+)= src[i]."""
    _run("scatter_rows", lambda: _native.check(_native.lib().dgc_scatter_rows(
        _p(src), _p(rows), _p(idx), n, width, _p(dst), int(add), _stream()), "dgc_scatter_rows"),
        n * (4 * width * (2 + int(add)) + 8))
    return dst


def softmax_xent(logits, labels, C, scale, dlogits, loss_partial, round_tf32=False,
                 dl_partial=None, dlogits16=None, scale16=1.0):
    """K8 dgc_softmax_xent; with dlogits16 (fp16 [n, C]) dgc_softmax_xent_f16,
    which also writes fp16(scale16 * dlogits) (dlogits may then be None)."""
    n = labels.numel()
    if dlogits16 is not None:
        _req16(dlogits16, "dlogits16")
        _run("softmax_xent", lambda: _native.check(_native.lib().dgc_softmax_xent_f16(
            _p(logits), _p(labels), n, C, float(scale), _p(dlogits), _p(loss_partial),
            _p(dl_partial), _p(dlogits16), float(scale16), _stream()), "dgc_softmax_xent_f16"),
            n * (6 * C + 4))
        return
    _run("softmax_xent", lambda: _native.check(_native.lib().dgc_softmax_xent(
        _p(logits), _p(labels), n, C, float(scale), int(round_tf32), _p(dlogits),
        _p(loss_partial), _p(dl_partial), _stream()), "dgc_softmax_xent"), n * (8 * C + 4))


def zero_(t):
    """dgc_zero_async: t = 0 by cudaMemsetAsync on the current stream (a memset
    node in a captured step instead of a torch fill kernel)."""
    _native.check(_native.lib().dgc_zero_async(_p(t), t.numel() * t.element_size(), _stream()),
                  "dgc_zero_async")


def readout_f16_grid(n):
    """CTAs (= rows of the dWo partial) of dgc_readout_f16 for n instances."""
    return int(_native.lib().dgc_readout_f16_grid(int(n)))


def readout_f16(h16, Wo16, bo, labels, C, scale, scale16, dh16, loss_partial, dl_partial,
                dwo_partial):
    """Fused fp16 readout (dgc_readout_f16): logits = h16 Wo16 + bo, softmax
    cross-entropy, S dh = (S dlogits16) Wo16^T as fp16, loss and bo partials per
    (128-row tile, TMEM lane quadrant) [4 ceil(n/128)], per-CTA dWo partials --
    one tcgen05 launch."""
    n, H = h16.shape
    _req16(h16, "h16"); _req16(Wo16, "Wo16"); _req16(dh16, "dh16")
    _req(bo, torch.float32, "bo"); _req(labels, torch.int32, "labels")
    _req(loss_partial, torch.float64, "loss_partial"); _req(dl_partial, torch.float32, "dl_partial")
    _req(dwo_partial, torch.float32, "dwo_partial")
    tiles, grid = 4 * ((n + 127) // 128), readout_f16_grid(n)  # partial rows per (tile, quadrant)
    if loss_partial.numel() < tiles or dl_partial.numel() < tiles * C or dwo_partial.numel() < grid * H * C:
        raise ValueError("readout_f16: partial buffers too small")
    # h16 read once, dh16 written, labels; the weights once per CTA
    nb = n * (2 * H + 2 * H + 4) + grid * (2 * H * C + 4 * H * C) + tiles * (8 + 4 * C)
    _run("readout_f16", lambda: _native.check(_native.lib().dgc_readout_f16(
        _p(h16), _p(Wo16), _p(bo), _p(labels), n, H, C, float(scale), float(scale16), _p(dh16),
        _p(loss_partial), _p(dl_partial), _p(dwo_partial), _stream()), "dgc_readout_f16"),
        nb, 2.0 * n * H * C * 3)


def readout_f16_evolve(h2_16, Wo16, bo, labels, C, scale, scale16, dz2, b2_partial, loss_partial,
                       dl_partial, dwo_partial):
    """dgc_readout_f16_evolve: the fused readout of EvolveGCN-O (input H2 =
    relu(.)): dz2 = dh * (H2 > 0) as fp32 and its column-sum partials (the b2
    gradient) instead of S dh16."""
    n, H = h2_16.shape
    _req16(h2_16, "h2_16"); _req16(Wo16, "Wo16"); _req(dz2, torch.float32, "dz2")
    _req(b2_partial, torch.float32, "b2_partial")
    _req(bo, torch.float32, "bo"); _req(labels, torch.int32, "labels")
    _req(loss_partial, torch.float64, "loss_partial"); _req(dl_partial, torch.float32, "dl_partial")
    _req(dwo_partial, torch.float32, "dwo_partial")
    tiles, grid = 4 * ((n + 127) // 128), readout_f16_grid(n)
    if (loss_partial.numel() < tiles or dl_partial.numel() < tiles * C or b2_partial.numel() < tiles * H
            or dwo_partial.numel() < grid * H * C):
        raise ValueError("readout_f16_evolve: partial buffers too small")
    nb = n * (2 * H + 4 * H + 4) + grid * (2 * H * C + 4 * H * C) + tiles * (8 + 4 * C + 4 * H)
    _run("readout_f16", lambda: _native.check(_native.lib().dgc_readout_f16_evolve(
        _p(h2_16), _p(Wo16), _p(bo), _p(labels), n, H, C, float(scale), float(scale16), _p(dz2),
        _p(b2_partial), _p(loss_partial), _p(dl_partial), _p(dwo_partial), _stream()),
        "dgc_readout_f16_evolve"), nb, 2.0 * n * H * C * 3)


def pack_tf32x24(x: np.ndarray) -> np.ndarray:
    """Host side of the TF32 input pipeline: round fp32 values to TF32 (round to
    nearest, ties away: cvt.rna.tf32) and keep the top three bytes of each
    (the low byte is zero) -> uint8 [3 * x.size]."""
    u = np.ascontiguousarray(x, dtype=np.float32).reshape(-1).view(np.uint32)
    finite = (u & np.uint32(0x7F800000)) != np.uint32(0x7F800000)
    r = np.where(finite, (u + np.uint32(0x1000)) & np.uint32(0xFFFFE000), u).astype(np.uint32)
    return np.ascontiguousarray(r.view(np.uint8).reshape(-1, 4)[:, 1:]).reshape(-1)


def unpack_tf32x24(packed, out):
    """dgc_unpack_tf32x24: out (fp32) from pack_tf32x24's 3-byte values."""
    _req(out, torch.float32, "out")
    n = out.numel()
    _run("unpack_tf32x24", lambda: _native.check(_native.lib().dgc_unpack_tf32x24(
        _p(packed), _p(out), n, _stream()), "dgc_unpack_tf32x24"), 7 * n)
    return out


def round_f16(x, out):
    """dgc_round_f16: out = fp32(RN_fp16(x)) (TF32 mode's in-range features)."""
    _run("round_f16", lambda: _native.check(_native.lib().dgc_round_f16(
        _p(x), _p(out), x.numel(), _stream()), "dgc_round_f16"), 8 * x.numel())
    return out


def unpack_f16(x16, out):
    """dgc_unpack_f16: out (fp32) = the fp16 features shipped from the host."""
    _req16(x16, "x16"); _req(out, torch.float32, "out")
    n = out.numel()
    _run("unpack_f16", lambda: _native.check(_native.lib().dgc_unpack_f16(
        _p(x16), _p(out), n, _stream()), "dgc_unpack_f16"), 6 * n)
    return out


def round_tf32(x, out):
    """dgc_round_tf32: out = RN_tf32(x)."""
    _run("round_tf32", lambda: _native.check(_native.lib().dgc_round_tf32(
        _p(x), _p(out), x.numel(), _stream()), "dgc_round_tf32"), 8 * x.numel())
    return out


def to_f16(x, out):
    """dgc_to_f16: out (fp16) = RN_fp16(x)."""
    _req(x, torch.float32, "x"); _req16(out, "out")
    _run("to_f16", lambda: _native.check(_native.lib().dgc_to_f16(
        _p(x), _p(out), x.numel(), _stream()), "dgc_to_f16"), 6 * x.numel())
    return out


def colsum(X, n, width, ld, out, scratch, accumulate=False):
    _run("colsum", lambda: _native.check(_native.lib().dgc_colsum(
        _p(X), n, width, ld, _p(out), int(accumulate), _p(scratch), _stream()), "dgc_colsum"),
        4 * n * width, n * width, 2)
    return out


def relu_bwd(dH, H, dZ):
    _run("relu_bwd", lambda: _native.check(_native.lib().dgc_relu_bwd(
        _p(dH), _p(H), _p(dZ), dH.numel(), _stream()), "dgc_relu_bwd"), 12 * dH.numel())
    return dZ


def sgd(p, g, mom, lr, momentum):
    _run("sgd", lambda: _native.check(_native.lib().dgc_sgd(
        _p(p), _p(g), _p(mom), p.numel(), float(lr), float(momentum), _stream()), "dgc_sgd"),
        20 * p.numel())


def adam_mirror(p, g, m, v, lr, b1, b2, eps, step, p_r=None, p16=None):
    """dgc_adam_dev_mirror: Adam (device step count) + the TF32 / fp16 parameter
    mirrors (p_r = rna_tf32(p), p16 = fp16(p_r)) in one launch."""
    _req(step, torch.int32, "step"); _req(p_r, torch.float32, "p_r"); _req16(p16, "p16")
    _run("adam", lambda: _native.check(_native.lib().dgc_adam_dev_mirror(
        _p(p), _p(g), _p(m), _p(v), p.numel(), float(lr), float(b1), float(b2), float(eps),
        _p(step), _p(p_r), _p(p16), _stream()), "dgc_adam_dev_mirror"),
        (28 + 4 * int(p_r is not None) + 2 * int(p16 is not None)) * p.numel())


def epoch_finish(loss_partial, loss_out, step=None):
    """dgc_epoch_finish: loss_out[0] = fixed-order sum of loss_partial (fp64);
    step (int32 CUDA tensor) += 1 when given."""
    _req(loss_partial, torch.float64, "loss_partial"); _req(loss_out, torch.float64, "loss_out")
    _req(step, torch.int32, "step")
    _run("epoch_finish", lambda: _native.check(_native.lib().dgc_epoch_finish(
        _p(loss_partial), loss_partial.numel(), _p(loss_out), _p(step), _stream()),
        "dgc_epoch_finish"), 8 * loss_partial.numel())


def adam(p, g, m, v, lr, b1, b2, eps, step):
    """dgc_adam (host step count) or dgc_adam_dev (step: int32 CUDA tensor)."""
    if isinstance(step, torch.Tensor):
        _req(step, torch.int32, "step")
        _run("adam", lambda: _native.check(_native.lib().dgc_adam_dev(
            _p(p), _p(g), _p(m), _p(v), p.numel(), float(lr), float(b1), float(b2), float(eps),
            _p(step), _stream()), "dgc_adam_dev"), 28 * p.numel())
        return
    _run("adam", lambda: _native.check(_native.lib().dgc_adam(
        _p(p), _p(g), _p(m), _p(v), p.numel(), float(lr), float(b1), float(b2), float(eps),
        int(step), _stream()), "dgc_adam"), 28 * p.numel())
