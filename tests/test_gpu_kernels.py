"""GPU parity of the individual kernels, called through the C ABI.
Float kernels are checked against a plain fp64 reference; the GRU and the
stale filter against the golden vectors the unmodified reference produced."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

dev = "cuda"


def t(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=dev)


def close(got, ref, rtol, what=""):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    scale = max(1e-30, float(np.abs(ref).max()))
    err = float(np.abs(got - ref).max()) / scale
    assert err <= rtol, f"{what}: max |err|/max|ref| = {err:.3e} > {rtol}"


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("prec,tol", [(3, 2e-6), (1, 2e-3)])
@pytest.mark.parametrize("M,N,K", [(1000, 16, 16), (777, 48, 16), (640, 128, 128),
                                   (300, 384, 128), (129, 64, 40), (5000, 512, 128)])
def test_gemm_tf32(a_mn, b_mn, prec, tol, M, N, K):
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    # TMA needs 16-byte row strides: pad the leading dimension of transposed copies
    def padded(x):
        ld = (x.shape[1] + 3) // 4 * 4
        out = np.zeros((x.shape[0], ld), np.float32)
        out[:, :x.shape[1]] = x
        return t(out), ld
    Ad, lda = padded(A.T) if a_mn else padded(A)
    Bd, ldb = padded(B) if b_mn else padded(B.T)
    C = torch.full((M, N), 7.0, device=dev)
    ops.gemm(Ad, Bd, C, M, N, K, a_mn=a_mn, b_mn=b_mn, lda=lda, ldb=ldb, precision=prec)
    close(C.cpu().numpy(), ref, tol, f"gemm a_mn={a_mn} b_mn={b_mn} p={prec}")


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("M,N,K", [(1000, 64, 64), (777, 128, 128), (300, 512, 128),
                                   (129, 64, 200), (5000, 256, 512)])
def test_gemm_f16(a_mn, b_mn, M, N, K):
    """K2 with fp16 operands (kind::f16; K-major and MN-major SWIZZLE_128B
    boxes) against fp64 of the same fp16-rounded operands; alpha = 2^-12 undoes
    a 2^12 operand scale exactly."""
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(M + N + K + 7)
    A = rng.standard_normal((M, K)).astype(np.float16)
    B = (rng.standard_normal((K, N)) * 4096).astype(np.float16)  # S-scaled operand
    ref = (A.astype(np.float64) @ B.astype(np.float64)) / 4096

    def padded(x):
        ld = (x.shape[1] + 7) // 8 * 8
        out = np.zeros((x.shape[0], ld), np.float16)
        out[:, :x.shape[1]] = x
        return t(out, torch.float16), ld
    Ad, lda = padded(A.T) if a_mn else padded(A)
    Bd, ldb = padded(B) if b_mn else padded(B.T)
    C = torch.full((M, N), 7.0, device=dev)
    ops.gemm_f16(Ad, Bd, C, M, N, K, a_mn=a_mn, b_mn=b_mn, lda=lda, ldb=ldb, alpha=2.0 ** -12)
    close(C.cpu().numpy(), ref, 1e-5, f"gemm_f16 a_mn={a_mn} b_mn={b_mn}")


def test_gemm_f16_fp16_outputs_and_mask():
    """fp16-only output (C16 = fp16(S * C), no fp32 C) with an fp16 ReLU-mask
    source and column sums, against fp64; and the same with an fp32 C beside."""
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(23)
    M, N, K, S = 1000, 128, 128, 4096.0
    A = (rng.standard_normal((M, K)) * S * 1e-4).astype(np.float16)   # an S-scaled gradient
    B = rng.standard_normal((N, K)).astype(np.float16)                # [N, K]: K-major B
    mask16 = rng.standard_normal((M, N)).astype(np.float16)
    ref = (A.astype(np.float64) @ B.astype(np.float64).T) / S * (mask16 > 0)
    C16 = torch.zeros((M, N), dtype=torch.float16, device=dev)
    cs = torch.zeros(((M + 127) // 128 * 4) * N, device=dev)
    ops.gemm_f16(t(A, torch.float16), t(B, torch.float16), None, M, N, K, b_mn=False, ldb=K,
                 alpha=1 / S, relu16=t(mask16, torch.float16), colsum_partial=cs, C16=C16,
                 c16_scale=S)
    torch.cuda.synchronize()
    close(C16.float().cpu().numpy() / S, ref, 2e-3, "fp16-only output")
    close(cs.view(-1, N).sum(0).cpu().numpy(), ref.sum(0), 1e-5, "column sums")
    C = torch.zeros((M, N), device=dev)
    ops.gemm_f16(t(A, torch.float16), t(B, torch.float16), C, M, N, K, b_mn=False, ldb=K,
                 alpha=1 / S, relu16=t(mask16, torch.float16))
    torch.cuda.synchronize()
    close(C.cpu().numpy(), ref, 1e-5, "fp32 output, fp16 mask")


def test_spmm_fp16_operand_and_outputs():
    """dgc_spmm_csr_h (fp16 gathered rows) equals the fp32 kernel on the same
    fp16 values bitwise; fp16 outputs = fp16(scale16 * out), with or without out."""
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(31)
    n, nc, W = 5000, 6000, 128
    deg = rng.integers(1, 20, n)
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(nc, d, replace=False)) for d in deg]).astype(np.int32)
    dinv = t(rng.random(nc).astype(np.float32) + 0.1)
    Y16 = t(rng.standard_normal((nc, W)).astype(np.float16), torch.float16)
    b = t(rng.standard_normal(W).astype(np.float32))
    ref = torch.zeros((n, W), device=dev)
    ops.spmm_csr(t(rp, torch.int32), t(col, torch.int32), dinv, Y16.float(), b, ref, act=1)
    out = torch.zeros((n, W), device=dev)
    o16 = torch.zeros((n, W), dtype=torch.float16, device=dev)
    ops.spmm_csr_h(t(rp, torch.int32), t(col, torch.int32), dinv, Y16, b, out, act=1, out16=o16,
                   scale16=8.0)
    torch.cuda.synchronize()
    assert torch.equal(out, ref) and torch.equal(o16, (ref * 8.0).half())
    o16b = torch.zeros_like(o16)
    ops.spmm_csr_h(t(rp, torch.int32), t(col, torch.int32), dinv, Y16, b, None, act=1, out16=o16b,
                   scale16=8.0)
    o16c = torch.zeros_like(o16)
    ops.spmm_csr(t(rp, torch.int32), t(col, torch.int32), dinv, Y16.float(), b, None, act=1,
                 out16=o16c, scale16=8.0)
    torch.cuda.synchronize()
    assert torch.equal(o16b, o16) and torch.equal(o16c, o16)


def test_gemm_f16_stacked_split_k():
    """[dWx; dU] = [x; h_in]^T (S dgx) with fp16 operands, split-K, alpha = 1/S:
    the BPTT weight-gradient form (MN-major A halves with their own strides)."""
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(11)
    n, F, H, S = 20000, 128, 128, 2.0 ** 16
    x = rng.standard_normal((n, F)).astype(np.float16)
    hs = np.zeros((n, 3 * H), np.float16)          # h_in inside a wider save row
    hs[:, :H] = rng.standard_normal((n, H)).astype(np.float16)
    dgx = (rng.standard_normal((n, 4 * H)) * 1e-5 * S).astype(np.float16)
    ref = np.concatenate([x, hs[:, :H]], 1).astype(np.float64).T @ dgx.astype(np.float64) / S
    C = torch.zeros((F + H, 4 * H), device=dev)
    splits = ops.gemm_splits(n, 2, 64)
    part = torch.zeros(splits * (F + H) * 4 * H, device=dev)
    ops.gemm_f16_stacked_a(t(x, torch.float16), t(hs, torch.float16), t(dgx, torch.float16), C, F,
                           F + H, 4 * H, n, a_mn=True, b_mn=True, lda0=F, lda1=3 * H, alpha=1 / S,
                           k_splits=64, partial=part)
    close(C.cpu().numpy(), ref, 1e-5, "stacked f16")


@pytest.mark.parametrize("splits", [1, 7, 64])
def test_gemm_split_k_weight_gradient(splits):
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(5)
    n, F, H = 20000, 128, 96
    X = rng.standard_normal((n, F)).astype(np.float32)
    dY = rng.standard_normal((n, H)).astype(np.float32)
    ref = X.astype(np.float64).T @ dY.astype(np.float64)
    C = torch.zeros((F, H), device=dev)
    part = torch.zeros(ops.gemm_splits(n, 3, splits) * F * H, device=dev)
    ops.gemm(t(X), t(dY), C, F, H, n, a_mn=True, precision=3, k_splits=splits, partial=part)
    close(C.cpu().numpy(), ref, 5e-6, "split-K")
    # determinism: bitwise identical on rerun
    C2 = torch.zeros_like(C)
    ops.gemm(t(X), t(dY), C2, F, H, n, a_mn=True, precision=3, k_splits=splits, partial=part)
    assert torch.equal(C, C2)


def test_gemm_epilogues_and_strides():
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(6)
    M, N, K, ld = 700, 64, 32, 80
    A = rng.standard_normal((M, ld)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    bias = rng.standard_normal(N).astype(np.float32)
    relu = rng.standard_normal((M, N)).astype(np.float32)
    C0 = rng.standard_normal((M, N)).astype(np.float32)
    ref = (C0 + A[:, :K].astype(np.float64) @ B + bias) * (relu > 0)
    C = t(C0)
    ops.gemm(t(A), t(B), C, M, N, K, lda=ld, precision=3, bias=t(bias), relu_src=t(relu),
             accumulate=True)
    close(C.cpu().numpy(), ref, 2e-6, "epilogue")


@pytest.mark.parametrize("M,N,K", [(700, 64, 32), (1000, 128, 128), (333, 512, 128)])
@pytest.mark.parametrize("relu", [False, True])
def test_gemm_tma_store_epilogue(M, N, K, relu):
    """TMA-store epilogue (plain / bias / ReLU mask / fused column sums):
    C = relu_mask(A B + bias); colsum partials reduce to the column sums of C."""
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(M + N + int(relu))
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    bias = rng.standard_normal(N).astype(np.float32)
    mask = rng.standard_normal((M, N)).astype(np.float32)
    ref = A.astype(np.float64) @ B + bias
    if relu:
        ref = ref * (mask > 0)
    C = torch.full((M, N), 3.0, device=dev)
    tiles = (M + 127) // 128
    cs = torch.zeros((4 * tiles, N), device=dev)
    ops.gemm(t(A), t(B), C, M, N, K, precision=3, bias=t(bias),
             relu_src=t(mask) if relu else None, colsum_partial=cs)
    close(C.cpu().numpy(), ref, 2e-6, "tma-store epilogue")
    out = torch.zeros(N, device=dev)
    ops.reduce_rows(cs, 4 * tiles, N, out)
    close(out.cpu().numpy(), ref.sum(0), 2e-5, "fused column sums")


@pytest.mark.parametrize("prec,tol", [(3, 5e-6), (1, 2e-3)])
def test_gemm_stacked_a(prec, tol):
    """[dWx; dU] = [x; h_in]^T dgx in one launch (two A operands with their own
    row strides), split-K, vs fp64."""
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(11)
    n, H, G = 20000, 128, 4
    X = rng.standard_normal((n, 2 * H)).astype(np.float32)     # x with ld 2H (an h|c buffer)
    S = rng.standard_normal((n, 7 * H)).astype(np.float32)     # save, h_in in the first H
    dG = rng.standard_normal((n, G * H)).astype(np.float32)
    ref = np.concatenate([X[:, :H].astype(np.float64).T @ dG, S[:, :H].astype(np.float64).T @ dG])
    C = torch.zeros((2 * H, G * H), device=dev)
    part = torch.zeros(ops.gemm_splits(n, prec, 96) * 2 * H * G * H, device=dev)
    ops.gemm_stacked_a(t(X), t(S), t(dG), C, H, 2 * H, G * H, n, a_mn=True, lda0=2 * H,
                       lda1=7 * H, ldb=G * H, ldc=G * H, precision=prec, k_splits=96, partial=part)
    close(C.cpu().numpy(), ref, tol, "stacked A")


def _csr(n_rows, n_cols, rng, max_deg=40):
    deg = rng.integers(0, max_deg, size=n_rows)
    deg[rng.random(n_rows) < 0.2] = 0
    rp = np.concatenate([[0], np.cumsum(deg + 1)]).astype(np.int32)
    col = []
    for i, d in enumerate(deg):
        c = np.sort(np.concatenate([[i], rng.choice(n_cols, size=d)]))
        col.append(c)
    return rp, np.concatenate(col).astype(np.int32)


@pytest.mark.parametrize("W", [16, 128, 512])
def test_spmm_csr(W):
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(W)
    n_rows, n_cols = 3000, 3500
    rp, col = _csr(n_rows, n_cols, rng)
    dinv = rng.random(n_cols).astype(np.float32) + 0.1
    Y = rng.standard_normal((n_cols, W)).astype(np.float32)
    b = rng.standard_normal(W).astype(np.float32)
    ref = np.zeros((n_rows, W))
    for i in range(n_rows):
        cs = col[rp[i]:rp[i + 1]]
        ref[i] = dinv[i] * (dinv[cs, None].astype(np.float64) * Y[cs]).sum(0) + b
    out = torch.zeros((n_rows, W), device=dev)
    ops.spmm_csr(t(rp, torch.int32), t(col, torch.int32), t(dinv), t(Y), t(b), out, act=1)
    close(out.cpu().numpy(), np.maximum(ref, 0), 1e-6, "spmm relu")
    ops.spmm_csr(t(rp, torch.int32), t(col, torch.int32), t(dinv), t(Y), None, out, act=0)
    close(out.cpu().numpy(), ref - b, 1e-6, "spmm")


def test_gru_forward_masked_matches_reference_golden(golden_dir):
    """Golden vectors of the reference gru_forward_masked (fusion.py:428-469),
    fp32 GPU vs fp64 reference within allclose(rtol=1e-4, atol=1e-6*max|ref|)
    (SURVEY.md §8(c) parity metric)."""
    from paper_2309_03523_b200.fusion import GruCell, gru_forward_masked, pack_sequences
    z = np.load(golden_dir / "gru.npz")
    for ci in range(4):
        p = f"c{ci}_"
        cell = GruCell(*(z[p + k] for k in GruCell.__dataclass_fields__))
        lengths = z[p + "lengths"].tolist()
        xs = z[p + "x"]
        offs = np.concatenate([[0], np.cumsum(lengths)])
        seqs = [(e, l) for e, l in enumerate(lengths)]
        inputs = {e: xs[offs[e]:offs[e + 1]] for e, _ in seqs}
        out = gru_forward_masked(cell, pack_sequences(seqs), inputs)
        got = np.concatenate([out[e] for e, _ in seqs])
        ref = z[p + "h"]
        np.testing.assert_allclose(got, ref, rtol=1e-4, atol=1e-6 * np.abs(ref).max())


def test_stale_filter_matches_reference_golden(golden_dir):
    """K5 against filter_transmissions/threshold on the reference DriftStream:
    identical send sets except keys inside the fp32-vs-fp64 tie band."""
    from paper_2309_03523_b200 import stale as st
    z = np.load(golden_dir / "stale.npz")
    modes = {"static3": st.StaleConfig.static(0.3), "tighten": st.StaleConfig.adaptive(True),
             "relax": st.StaleConfig.adaptive(), "off": st.StaleConfig.off()}
    for name, cfg in modes.items():
        emb, send, theta_ref = z[name + "_emb"], z[name + "_send"], z[name + "_theta"]
        n, dim = emb.shape[1:]
        cache = st.EmbeddingCacheGPU(n, dim, dev)
        trace = st.EpochLossTrace()
        for r in range(1, emb.shape[0] + 1):
            keys = np.arange(n)[(np.arange(n) + r) % 4 != 0]
            Y = t(emb[r - 1])
            # the reference cache is keyed by instance: emulate with all n keys
            # but only the boundary subset participates this epoch
            sub = st.EmbeddingCacheGPU(len(keys), dim, dev)
            sub.values.copy_(cache.values[t(keys, torch.long)])
            sub.cached.copy_(cache.cached[t(keys, torch.long)])
            kr = t(keys, torch.int32)
            theta = 0.0
            if r >= 2:
                dmax = st.cache_gap_gpu(Y, kr, sub)
                d_r = float(dmax.item())
                theta = st.threshold(trace, r, d_r, cfg)
                assert theta == pytest.approx(theta_ref[r - 1], rel=1e-6)
            s = st.filter_transmissions_gpu(Y, kr, sub, theta).cpu().numpy().astype(bool)
            got = np.zeros(n, np.uint8)
            got[keys[s]] = 1
            mism = np.flatnonzero(got != send[r - 1])
            if len(mism):
                dist = sub.dist.cpu().numpy()
                pos = np.searchsorted(keys, mism)
                assert np.all(np.abs(dist[pos] - theta) <= 1e-5 * max(theta, 1e-30)), name
            cache.values[t(keys, torch.long)] = sub.values
            cache.cached[t(keys, torch.long)] = sub.cached
            trace.append(2.0 * 0.9 ** (r - 1))


@pytest.mark.parametrize("width,n_keys", [(64, 1001), (32, 4099), (16, 7), (128, 333),
                                          (256, 5), (12, 1003)])
def test_stale_distance_all_widths(width, n_keys):
    """K5 distance at every sub-warp width (LPR 1/8/32), including the LPR = 8
    path (widths 32-124: four keys per warp) with n_keys not a multiple of 4,
    against numpy fp64: distances, D_r = max over cached keys, and the send
    decision (the tail warp used to shuffle unconverged)."""
    from paper_2309_03523_b200 import stale as st
    rng = np.random.default_rng(width + n_keys)
    n_rows = n_keys + 50
    Y = rng.standard_normal((n_rows, width)).astype(np.float32)
    keys = rng.permutation(n_rows)[:n_keys].astype(np.int32)
    cache = st.EmbeddingCacheGPU(n_keys, width, dev)
    cv = (Y[keys] + 0.1 * rng.standard_normal((n_keys, width))).astype(np.float32)
    cached = (rng.random(n_keys) < 0.8).astype(np.uint8)
    cache.values.copy_(t(cv))
    cache.cached.copy_(t(cached, torch.uint8))
    dmax = float(st.cache_gap_gpu(t(Y), t(keys, torch.int32), cache).item())
    ref = np.sqrt(((Y[keys].astype(np.float64) - cv) ** 2).sum(axis=1))
    np.testing.assert_allclose(cache.dist.cpu().numpy(), ref, rtol=1e-5)
    assert dmax == pytest.approx(ref[cached.astype(bool)].max(), rel=1e-5)
    theta = float(np.median(ref))
    s = st.filter_transmissions_gpu(t(Y), t(keys, torch.int32), cache, theta).cpu().numpy()
    exp = (~cached.astype(bool)) | (cache.dist.cpu().numpy() > theta)
    np.testing.assert_array_equal(s.astype(bool), exp)


def test_exchange_pack_unpack():
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(9)
    n_keys, W = 5000, 16
    pos = np.sort(rng.choice(n_keys, 3000, replace=False)).astype(np.int32)
    send = (rng.random(n_keys) < 0.3).astype(np.uint8)
    out = torch.zeros(3000, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    ops.compact_sent(t(pos, torch.int32), t(send, torch.uint8), out, cnt)
    ref = np.flatnonzero(send[pos])
    c = int(cnt.item())
    assert c == len(ref)
    np.testing.assert_array_equal(out[:c].cpu().numpy(), ref)
    Y = rng.standard_normal((n_keys, W)).astype(np.float32)
    rows = rng.permutation(n_keys)[:3000].astype(np.int32)
    buf = torch.zeros((c, W), device=dev)
    ops.gather_rows(t(Y), t(rows, torch.int32), out[:c], c, W, buf)
    np.testing.assert_array_equal(buf.cpu().numpy(), Y[rows[ref]])
    dst = torch.zeros((n_keys, W), device=dev)
    ops.scatter_rows(buf, t(rows, torch.int32), out[:c], c, W, dst, add=True)
    ops.scatter_rows(buf, t(rows, torch.int32), out[:c], c, W, dst, add=True)
    exp = np.zeros((n_keys, W), np.float32)
    exp[rows[ref]] = 2 * Y[rows[ref]]
    np.testing.assert_array_equal(dst.cpu().numpy(), exp)


@pytest.mark.parametrize("W,stale", [(16, True), (128, True), (64, False), (8, True)])
def test_exchange_data_plane(W, stale):
    """One-buffer exchange (csrc/exchange.cu) for D = 4 virtual devices vs
    numpy: device compaction of every peer's list, records, unpack into halo
    rows, reverse pack of the fresh rows' gradients and the fixed-order
    add-back (ascending peer)."""
    from paper_2309_03523_b200 import ops
    from paper_2309_03523_b200.trainer import ExchangePlan
    rng = np.random.default_rng(W)
    D, me, n_keys, n_own = 4, 1, 700, 2000
    key_rows = np.sort(rng.choice(n_own, n_keys, replace=False)).astype(np.int32)
    lists = [np.sort(rng.choice(n_keys, int(rng.integers(0, 400)), replace=False)) if p != me
             else np.zeros(0, np.int64) for p in range(D)]
    send_ptr = np.cumsum([0] + [len(l) for l in lists])
    send_pos = np.concatenate(lists).astype(np.int32)
    halo_owner = rng.integers(0, D, 900)  # every halo row has one owner (disjoint lists)
    rl = [np.flatnonzero((halo_owner == p) & (rng.random(900) < 0.7)) + n_own if p != me
          else np.zeros(0, np.int64) for p in range(D)]
    recv_ptr = np.cumsum([0] + [len(l) for l in rl])
    recv_slot = np.concatenate(rl).astype(np.int32)
    xp = ExchangePlan(D, send_ptr, send_pos, recv_ptr, recv_slot, W, dev, n_keys)
    Y = rng.standard_normal((n_own + 900, W)).astype(np.float32)
    send = (rng.random(n_keys) < 0.6).astype(np.uint8) if stale else np.ones(n_keys, np.uint8)
    slot = None
    if stale:
        ops.exchange_rank(xp.ent_key, xp.ent_ptr, D, t(send, torch.uint8), xp.ent_slot, xp.counts)
        slot = xp.ent_slot
    Yt = t(Y)
    ops.exchange_pack(Yt, W, t(key_rows, torch.int32), xp.ent_key, xp.ent_idx, slot, xp.sendbuf)
    cnt = xp.counts.cpu().numpy()
    rec = xp.sendbuf.cpu().numpy()
    o = 0
    for p in range(D):
        sel = [j for j, k in enumerate(lists[p]) if send[k]]
        assert cnt[p] == len(sel)
        for j in sel:
            r = rec[o * (W + 4):(o + 1) * (W + 4)]
            assert r[:1].view(np.int32)[0] == j
            np.testing.assert_array_equal(r[4:], Y[key_rows[lists[p][j]]])
            o += 1
    # receive: records from the peers for my recv lists (every other fresh)
    rcnt = np.zeros(D, np.int32)
    recs, fresh = [], []
    for p in range(D):
        js = [j for j in range(len(rl[p])) if j % 2 == 0]
        rcnt[p] = len(js)
        for j in js:
            v = rng.standard_normal(W).astype(np.float32)
            recs.append(np.concatenate([np.asarray([j, 0, 0, 0], np.int32).view(np.float32), v]))
            fresh.append((rl[p][j], v))
    rbuf = t(np.concatenate(recs) if recs else np.zeros(W + 4, np.float32))
    dst = Yt.clone()
    ops.exchange_unpack(rbuf, W, t(rcnt, torch.int32), D, xp.rlist, xp.rlist_ptr, len(recs), dst)
    exp = Y.copy()
    for s_, v in fresh:
        exp[s_] = v
    np.testing.assert_array_equal(dst.cpu().numpy(), exp)
    # reverse: gradient rows of the fresh halo rows, in received order
    dY = rng.standard_normal((n_own + 900, W)).astype(np.float32)
    back = torch.zeros(max(1, len(recs)) * W, device=dev)
    ops.exchange_pack_back(rbuf, W, t(rcnt, torch.int32), D, xp.rlist, xp.rlist_ptr, len(recs),
                           t(dY), back)
    np.testing.assert_array_equal(back.cpu().numpy()[:len(recs) * W].reshape(-1, W),
                                  np.asarray([dY[s_] for s_, _ in fresh]).reshape(-1, W))
    # add-back: the gradients returned for my sent records, fixed peer order
    n_sent = int(cnt.sum())
    g = rng.standard_normal((max(1, n_sent), W)).astype(np.float32)
    dYt = t(dY)
    ops.exchange_add_back(t(g), W, t(key_rows, torch.int32), xp.kent_ptr, xp.kent, slot, dYt)
    exp = dY.copy()
    acc = {}
    o = 0
    for p in range(D):
        for j, k in enumerate(lists[p]):
            if send[k]:
                acc.setdefault(int(k), []).append(g[o])
                o += 1
    for k, gs in acc.items():
        v = exp[key_rows[k]].copy()
        for x in gs:  # ascending peer
            v = v + x
        exp[key_rows[k]] = v
    np.testing.assert_array_equal(dYt.cpu().numpy(), exp)


def test_spmm_row_subsets_equal_full():
    """dgc_spmm_csr_rows on interior / boundary row lists and on row ranges
    is bitwise the full dgc_spmm_csr."""
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(3)
    n, nc, W = 3000, 3500, 128
    deg = rng.integers(1, 30, n)
    row_ptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(nc, d, replace=False)) for d in deg]).astype(np.int32)
    dinv = rng.random(nc).astype(np.float32)
    Y = t(rng.standard_normal((nc, W)).astype(np.float32))
    b = t(rng.standard_normal(W).astype(np.float32))
    full = torch.zeros((n, W), device=dev)
    ops.spmm_csr(t(row_ptr, torch.int32), t(col, torch.int32), t(dinv), Y, b, full, act=1)
    bnd = np.asarray([(col[row_ptr[i]:row_ptr[i + 1]] >= n).any() for i in range(n)])
    part = torch.zeros((n, W), device=dev)
    for rows in (np.flatnonzero(~bnd), np.flatnonzero(bnd)):
        ops.spmm_csr_rows(t(row_ptr, torch.int32), t(col, torch.int32), t(dinv), Y, b, part, act=1,
                          rows=t(rows, torch.int32))
    assert torch.equal(part, full)
    part.zero_()
    ops.spmm_csr_rows(t(row_ptr, torch.int32), t(col, torch.int32), t(dinv), Y, b, part, act=1,
                      n_rows=1234, row_begin=n - 1234)
    ops.spmm_csr_rows(t(row_ptr, torch.int32), t(col, torch.int32), t(dinv), Y, b, part, act=1,
                      n_rows=n - 1234, row_begin=0)
    assert torch.equal(part, full)
    # dynamic row scheduling (work counter; 2.5M rows of width 128 so that every
    # resident warp has >= 256 rows and the dynamic path runs): bitwise the
    # static result, and the counter pair is left zeroed for the next launch
    work = torch.zeros(2, dtype=torch.int32, device=dev)
    nb = 148 * 64 * 256 + 3333
    deg2 = rng.integers(1, 6, nb)
    rp2 = np.concatenate([[0], np.cumsum(deg2)]).astype(np.int32)
    c2 = np.sort(rng.integers(0, nb, (nb, 5)), 1)[np.arange(5)[None, :] < deg2[:, None]].astype(np.int32)
    d2 = t(rng.random(nb).astype(np.float32))
    Y2 = torch.randn((nb, W), device=dev)
    st, dy = torch.zeros((nb, W), device=dev), torch.zeros((nb, W), device=dev)
    ops.spmm_csr(t(rp2, torch.int32), t(c2, torch.int32), d2, Y2, None, st, act=0)
    for _ in range(2):
        ops.spmm_csr(t(rp2, torch.int32), t(c2, torch.int32), d2, Y2, None, dy, act=0, work=work)
        assert torch.equal(st, dy) and work.cpu().tolist() == [0, 0]
    for _ in range(3):
        dyn = torch.zeros((n, W), device=dev)
        ops.spmm_csr(t(row_ptr, torch.int32), t(col, torch.int32), t(dinv), Y, b, dyn, act=1,
                     work=work)
        assert torch.equal(dyn, full)
        assert work.cpu().tolist() == [0, 0]
    part.zero_()
    for rows in (np.flatnonzero(~bnd), np.flatnonzero(bnd)):
        ops.spmm_csr_rows(t(row_ptr, torch.int32), t(col, torch.int32), t(dinv), Y, b, part, act=1,
                          rows=t(rows, torch.int32), work=work)
    assert torch.equal(part, full) and work.cpu().tolist() == [0, 0]


def test_softmax_xent_colsum_optimizers():
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(10)
    n, C = 3001, 16
    logits = rng.standard_normal((n, C)).astype(np.float32) * 3
    y = rng.integers(0, C, n).astype(np.int32)
    dl = torch.zeros((n, C), device=dev)
    lp = torch.zeros((n + 255) // 256, dtype=torch.float64, device=dev)
    ops.softmax_xent(t(logits), t(y, torch.int32), C, 0.5, dl, lp)
    x = logits.astype(np.float64)
    m = x.max(1, keepdims=True)
    logp = x - m - np.log(np.exp(x - m).sum(1, keepdims=True))
    assert float(lp.sum()) == pytest.approx(-logp[np.arange(n), y].sum(), rel=1e-5)
    g = np.exp(logp)
    g[np.arange(n), y] -= 1
    close(dl.cpu().numpy(), 0.5 * g, 1e-5, "dlogits")
    out = torch.zeros(C, device=dev)
    scratch = torch.zeros(296 * C, device=dev)
    ops.colsum(t(logits), n, C, C, out, scratch)
    close(out.cpu().numpy(), x.sum(0), 1e-5, "colsum")
    p = rng.standard_normal(1000).astype(np.float32)
    gr = rng.standard_normal(1000).astype(np.float32)
    pd, md, vd = t(p), torch.zeros(1000, device=dev), torch.zeros(1000, device=dev)
    ops.adam(pd, t(gr), md, vd, 0.01, 0.9, 0.999, 1e-8, 1)
    mm = 0.1 * gr
    vv = 0.001 * gr * gr
    ref = p - 0.01 * (mm / 0.1) / (np.sqrt(vv / 0.001) + 1e-8)
    close(pd.cpu().numpy(), ref, 1e-6, "adam")


def tc_save_decode(save, H):
    """The tensor-core LSTM save rows as [n, 6H] fp32 (h_in, c_in, i, f, g, o):
    the compact H = 128 cluster layout (fp16 h_in | c_in | i, f, g, o
    interleaved per unit, 3 H floats per row) or the 7 H fp32 layout."""
    from paper_2309_03523_b200 import ops
    save = np.ascontiguousarray(save, np.float32)
    sf = ops.rnn_tc_save_floats(H)
    if sf == 7 * H:
        return save[:, :6 * H]
    half = save[:, :sf].copy().view(np.float16).astype(np.float32)  # [n, 6H]
    n = save.shape[0]
    ifgo = half[:, 2 * H:].reshape(n, H, 4).transpose(0, 2, 1).reshape(n, 4 * H)
    return np.concatenate([half[:, :2 * H], ifgo], 1)


def tc_save_encode(fields, H):
    """Inverse of tc_save_decode for [n, 7H] fp32 inputs (tanh(c) dropped when compact)."""
    from paper_2309_03523_b200 import ops
    sf = ops.rnn_tc_save_floats(H)
    if sf == 7 * H:
        return np.ascontiguousarray(fields, np.float32)
    n = fields.shape[0]
    ifgo = fields[:, 2 * H:6 * H].reshape(n, 4, H).transpose(0, 2, 1).reshape(n, 4 * H)
    half = np.concatenate([fields[:, :2 * H], ifgo], 1).astype(np.float16)
    return np.ascontiguousarray(half).view(np.float32)


def run_end_rows(slot_row, mask):
    """Instances at the last slot of their run (next slot absent or not continuing)."""
    sr = np.asarray(slot_row).reshape(mask.shape)
    nxt = np.zeros_like(mask)
    nxt[:, :-1] = mask[:, 1:]
    return sr[(sr >= 0) & (nxt == 0)]


@pytest.mark.parametrize("H,ew16", [(32, False), (64, False), (128, False), (128, True)])
def test_lstm_fwd_tensor_core_matches_simt(H, ew16, monkeypatch):
    """K4 on tcgen05 (TF32) vs the fp32 SIMT kernel on the same packed runs,
    with cross-device carries at some run starts (ew16: the 16-epilogue-warp
    cluster variant used when rq > 24)."""
    if ew16:
        monkeypatch.setenv("DGC_RNN_EW16", "1")
    from paper_2309_03523_b200 import ops
    from paper_2309_03523_b200.layout import pack_sequences_native
    rng = np.random.default_rng(H)
    lengths = rng.integers(1, 20, size=700)
    seq, pos, mask, _ = pack_sequences_native(lengths)
    R, L = seq.shape
    offs = np.concatenate([[0], np.cumsum(lengths)])
    n = int(offs[-1])
    slot_row = np.where(seq >= 0, offs[np.maximum(seq, 0)] + pos, -1).astype(np.int32)
    run_carry = np.where(rng.random(len(lengths)) < 0.3, 1, -1)
    n_carry = int((run_carry > 0).sum())
    run_carry[run_carry > 0] = np.arange(n_carry)
    slot_carry = np.where((seq >= 0) & (pos == 0), run_carry[np.maximum(seq, 0)], -1).astype(np.int32)
    gx = rng.standard_normal((n, 4 * H)).astype(np.float32)
    U = (rng.standard_normal((H, 4 * H)) / np.sqrt(H)).astype(np.float32)
    carry = rng.standard_normal((max(n_carry, 1), 2 * H)).astype(np.float32)
    outs = []
    for tc in (False, True):
        hc = torch.zeros((n, 2 * H), device=dev)
        save = torch.zeros((n, ops.rnn_tc_save_floats(H) if tc else 7 * H), device=dev)
        args = (t(gx), None, t(slot_row.reshape(-1), torch.int32), t(mask.reshape(-1), torch.uint8),
                t(slot_carry.reshape(-1), torch.int32), t(carry), R, L, H, 2 * H, hc, hc[:, H:], save)
        if tc:
            Ut = t(U.T.copy())
            ops.rnn_fwd_tc(1, args[0], Ut, *args[2:])
        else:
            ops.rnn_fwd(1, args[0], t(U), *args[2:])
        torch.cuda.synchronize()
        sv = save.cpu().numpy()
        outs.append((hc.cpu().numpy(), tc_save_decode(sv, H) if tc else sv[:, :6 * H]))
    # the cluster forward (H = 128) writes c only at run ends (the carries)
    ends = run_end_rows(slot_row, mask)
    close(outs[1][0][:, :H], outs[0][0][:, :H], 2e-3, "lstm tc h")
    close(outs[1][0][ends, H:], outs[0][0][ends, H:], 2e-3, "lstm tc c at run ends")
    # h_in .. o (the H = 128 cluster forward stores no tanh(c): its BPTT recomputes
    # tanh(f c_in + i g), and keeps c_in, i, f, g, o in fp16)
    close(outs[1][1], outs[0][1], 2e-3, "lstm tc save")


@pytest.mark.parametrize("n_seq,carry_frac", [(700, 0.3), (9000, 0.0), (16000, 0.1)])
def test_lstm_fwd_fused_projection_matches_two_step(n_seq, carry_frac):
    """The fused-projection forward (fp16 x rows TMA-gathered by slot_row, x
    Wx^T + h U^T + b in TMEM from resident fp16 weights) equals gx = x Wx + b
    (K2) followed by the unfused TF32 tensor-core forward: h|c and every saved
    field (the operands are TF32-rounded, so their fp16 copies are exact; fp16
    and TF32 carry the same 10-bit mantissa). The fp16 copy of h_out is h_out.
    16000 sequences -> R > 7104 packed rows -> rq > 24 rows per lane quadrant
    (the 16-epilogue-warp variants)."""
    from paper_2309_03523_b200 import ops
    from paper_2309_03523_b200.layout import pack_sequences_native
    H = 128
    if not ops.rnn_fwd_tc_fused_available(H, H):
        pytest.skip("fused projection disabled in this process")
    rng = np.random.default_rng(n_seq)
    lengths = rng.integers(1, 20, size=n_seq)
    seq, pos, mask, _ = pack_sequences_native(lengths)
    R, L = seq.shape
    offs = np.concatenate([[0], np.cumsum(lengths)])
    n = int(offs[-1])
    # instances not in slot order: a random permutation of the rows
    perm = rng.permutation(n)
    slot_row = np.where(seq >= 0, perm[offs[np.maximum(seq, 0)] + pos], -1).astype(np.int32)
    run_carry = np.where(rng.random(len(lengths)) < carry_frac, 1, -1)
    n_carry = int((run_carry > 0).sum())
    run_carry[run_carry > 0] = np.arange(n_carry)
    slot_carry = np.where((seq >= 0) & (pos == 0), run_carry[np.maximum(seq, 0)], -1).astype(np.int32)
    rnd = lambda a: t(a)
    x = t(rng.standard_normal((n, 2 * H)).astype(np.float32))   # ld 2H, like an h|c buffer
    ops.round_tf32(x, x)
    Wx = t((rng.standard_normal((H, 4 * H)) / np.sqrt(H)).astype(np.float32)); ops.round_tf32(Wx, Wx)
    U = t((rng.standard_normal((H, 4 * H)) / np.sqrt(H)).astype(np.float32)); ops.round_tf32(U, U)
    b = t(rng.standard_normal(4 * H).astype(np.float32) * 0.1)
    carry = t(rng.standard_normal((max(n_carry, 1), 2 * H)).astype(np.float32))
    sr, sm, sc = t(slot_row.reshape(-1), torch.int32), t(mask.reshape(-1), torch.uint8), \
        t(slot_carry.reshape(-1), torch.int32)
    Ut = U.t().contiguous()
    outs = []
    for fused in (False, True):
        hc = torch.zeros((n, 2 * H), device=dev)
        save = torch.zeros((n, ops.rnn_tc_save_floats(H)), device=dev)
        if fused:
            h16 = torch.zeros((n, H), dtype=torch.float16, device=dev)
            ops.lstm_fwd_tc_f16x(x[:, :H].half(), Wx, U, b, sr, sm, sc, carry, R, L, H, 2 * H, hc,
                                 hc[:, H:], save, h_out16=h16)
            torch.cuda.synchronize()
            assert torch.equal(h16.float(), hc[:, :H])
            # fp32 h at run ends only: same fp16 output, same run-end rows, nothing else
            hc2 = torch.zeros_like(hc)
            h16b = torch.zeros_like(h16)
            ops.lstm_fwd_tc_f16x(x[:, :H].half(), Wx, U, b, sr, sm, sc, carry, R, L, H, 2 * H,
                                 hc2, hc2[:, H:], torch.zeros_like(save), h_out16=h16b,
                                 h32_run_ends_only=True)
            torch.cuda.synchronize()
            assert torch.equal(h16b, h16)
            ends_t = torch.as_tensor(run_end_rows(slot_row, mask), device=dev)
            inner = torch.ones(n, dtype=torch.bool, device=dev)
            inner[ends_t] = False
            assert torch.equal(hc2[ends_t], hc[ends_t]) and not hc2[inner, :H].any()
        else:
            gx = torch.zeros((n, 4 * H), device=dev)
            ops.gemm(x, Wx, gx, n, 4 * H, H, lda=2 * H, precision=1, bias=b)
            ops.rnn_fwd_tc(1, gx, Ut, sr, sm, sc, carry, R, L, H, 2 * H, hc, hc[:, H:], save)
        torch.cuda.synchronize()
        outs.append((hc.cpu().numpy(), save.cpu().numpy()))
    close(outs[1][0], outs[0][0], 2e-3, "fused h|c")  # TF32 operand rounding differs
    ends = run_end_rows(slot_row, mask)
    assert np.abs(outs[1][0][ends, H:]).max() > 0  # c written at every run end
    close(tc_save_decode(outs[1][1], H), tc_save_decode(outs[0][1], H), 2e-3, "fused save")


@pytest.mark.parametrize("H,variant,n_seq", [(32, "", 700), (64, "", 700), (128, "", 700),
                                             (128, "", 6900), (128, "ew16", 700),
                                             (128, "2sm", 700), (128, "2sm", 6900)])
def test_lstm_bwd_tensor_core_matches_simt(H, variant, n_seq, monkeypatch):
    """K4 BPTT on tcgen05 vs the fp32 SIMT BPTT on the same packed runs: dgx and
    the fused bias partial sums. H = 128: the K-split cluster kernel with 12 / 16
    (ew16) epilogue warps, or the opt-in 2-SM (cta_group::2) kernel (6900 runs:
    12 rows per lane quadrant, every epilogue warp busy)."""
    if variant == "2sm":
        monkeypatch.setenv("DGC_BPTT_2SM", "1")
    if variant == "ew16":
        monkeypatch.setenv("DGC_RNN_EW16", "1")
    from paper_2309_03523_b200 import ops
    from paper_2309_03523_b200.layout import pack_sequences_native
    rng = np.random.default_rng(H + 1)
    lengths = rng.integers(1, 20, size=n_seq)
    seq, pos, mask, _ = pack_sequences_native(lengths)
    R, L = seq.shape
    offs = np.concatenate([[0], np.cumsum(lengths)])
    n = int(offs[-1])
    slot_row = np.where(seq >= 0, offs[np.maximum(seq, 0)] + pos, -1).astype(np.int32).reshape(-1)
    U = (rng.standard_normal((H, 4 * H)) / np.sqrt(H)).astype(np.float32)
    save = np.concatenate([rng.standard_normal((n, 2 * H)),            # h_in, c_in
                           rng.random((n, 4 * H)),                      # i, f, g, o
                           np.zeros((n, H))], 1).astype(np.float32)
    ci, ig, fg, gg = (save[:, k * H:(k + 1) * H] for k in (1, 2, 3, 4))
    save[:, 6 * H:] = np.tanh(fg * ci + ig * gg)                       # tanh(c) of the forward
    dh = rng.standard_normal((n, H)).astype(np.float32)
    outs = []
    for tc in (False, True):
        dgx = torch.zeros((n, 4 * H), device=dev)
        sr, sm = t(slot_row, torch.int32), t(mask.reshape(-1), torch.uint8)
        if tc:
            tiles = ops.rnn_tc_tiles(R, H)
            bp = torch.zeros((tiles, 4 * H), device=dev)
            scr = torch.zeros(((R + 127) // 128 * 128, H), device=dev)
            ops.rnn_bwd_tc(1, t(U), sr, sm, R, L, H, t(tc_save_encode(save, H)), t(dh), dgx, scr,
                           bias_partial=bp)
            bias = bp.sum(0)
        else:
            rows = ops.rnn_bwd_partial_rows(R, H)
            bp = torch.zeros((rows, 4 * H), device=dev)
            ops.rnn_bwd(1, t(U.T.copy()), sr, sm, R, L, H, t(save), t(dh), dgx, bias_partial=bp)
            bias = bp.sum(0)
        torch.cuda.synchronize()
        outs.append((dgx.cpu().numpy(), bias.cpu().numpy()))
    close(outs[1][0], outs[0][0], 3e-3, "lstm bwd tc dgx")
    close(outs[1][1], outs[0][1], 3e-3, "lstm bwd tc bias")


@pytest.mark.parametrize("variant,dgx16", [("", False), ("", True), ("ew16", True)])
def test_lstm_bwd_tc_f16_dh_out_equals_fp32(variant, dgx16, monkeypatch):
    """K-split cluster BPTT with an S-scaled fp16 dh_out (cell bit 25, the fp16
    readout / input-gradient GEMMs' output) is bitwise the fp32-dh_out kernel
    fed the same values (fp16(S dh) / S is exact in fp32)."""
    if variant == "ew16":
        monkeypatch.setenv("DGC_RNN_EW16", "1")
    from paper_2309_03523_b200 import ops
    from paper_2309_03523_b200.layout import pack_sequences_native
    H, e = 128, 12
    rng = np.random.default_rng(5)
    lengths = rng.integers(1, 20, size=900)
    seq, pos, mask, _ = pack_sequences_native(lengths)
    R, L = seq.shape
    offs = np.concatenate([[0], np.cumsum(lengths)])
    n = int(offs[-1])
    slot_row = np.where(seq >= 0, offs[np.maximum(seq, 0)] + pos, -1).astype(np.int32).reshape(-1)
    U = (rng.standard_normal((H, 4 * H)) / np.sqrt(H)).astype(np.float32)
    save = np.concatenate([rng.standard_normal((n, 2 * H)), rng.random((n, 4 * H)),
                           np.zeros((n, H))], 1).astype(np.float32)
    dh16 = (rng.standard_normal((n, H)) / 64).astype(np.float16)  # S dh
    dh32 = dh16.astype(np.float32) / np.float32(2.0 ** e)
    sr, sm = t(slot_row, torch.int32), t(mask.reshape(-1), torch.uint8)
    sv = t(tc_save_encode(save, H))
    outs = []
    for d in (t(dh32), torch.as_tensor(dh16).to(dev)):
        dgx = torch.zeros((n, 4 * H), device=dev, dtype=torch.float16 if dgx16 else torch.float32)
        bp = torch.zeros((ops.rnn_tc_tiles(R, H), 4 * H), device=dev)
        scr = torch.zeros(((R + 127) // 128 * 128, H), device=dev)
        ops.rnn_bwd_tc(1 | (e << 16), t(U), sr, sm, R, L, H, sv, d, dgx, scr, bias_partial=bp)
        torch.cuda.synchronize()
        outs.append((dgx.float().cpu().numpy(), bp.cpu().numpy()))
    assert np.abs(outs[0][0]).max() > 0
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("n,C", [(300, 16), (5000, 16), (2049, 32), (40000, 16)])
def test_fused_readout_f16_matches_fp64(n, C):
    """dgc_readout_f16 (logits GEMM + softmax-xent + S dh + dWo in one tcgen05
    launch) vs an fp64 restatement on the same fp16 operands: loss, bo / Wo
    gradients and the S-scaled fp16 dh; ragged last tile and padding labels."""
    from paper_2309_03523_b200 import ops
    H, e = 128, 13
    S = 2.0 ** e
    rng = np.random.default_rng(n + C)
    h16 = rng.standard_normal((n, H)).astype(np.float16)
    Wo16 = (rng.standard_normal((H, C)) / np.sqrt(H)).astype(np.float16)
    bo = (0.1 * rng.standard_normal(C)).astype(np.float32)
    y = rng.integers(0, C, size=n).astype(np.int32)
    y[rng.random(n) < 0.1] = -1  # padding rows
    scale = 1.0 / n
    tiles, grid = 4 * ((n + 127) // 128), ops.readout_f16_grid(n)  # (tile, quadrant) rows
    dh16 = torch.zeros((n, H), device=dev, dtype=torch.float16)
    lp = torch.zeros(tiles, device=dev, dtype=torch.float64)
    dp = torch.zeros(tiles * C, device=dev)
    wp = torch.zeros(grid * H * C, device=dev)
    ops.readout_f16(torch.as_tensor(h16).to(dev), torch.as_tensor(Wo16).to(dev), t(bo),
                    t(y, torch.int32), C, scale, S, dh16, lp, dp, wp)
    gWo = torch.zeros(H * C, device=dev)
    gbo = torch.zeros(C, device=dev)
    ops.reduce_rows_batched([(dp, tiles, C, gbo), (wp, grid, H * C, gWo)])
    torch.cuda.synchronize()
    # fp64 reference on the same fp16 operands
    hd, Wd = h16.astype(np.float64), Wo16.astype(np.float64)
    z = hd @ Wd + bo.astype(np.float64)
    z -= z.max(1, keepdims=True)
    p = np.exp(z) / np.exp(z).sum(1, keepdims=True)
    real = y >= 0
    loss = -np.log(p[np.arange(n)[real], y[real]]).sum()
    dl = p.copy()
    dl[np.arange(n)[real], y[real]] -= 1.0
    dl[~real] = 0.0
    dl *= scale
    dl16 = (dl * S).astype(np.float16).astype(np.float64)
    dh_ref = dl16 @ Wd.T
    dWo_ref = hd.T @ dl16 / S
    assert abs(lp.sum().item() - loss) <= 1e-5 * abs(loss)
    close(gbo.cpu().numpy(), dl.sum(0), 1e-4, "bo grad")
    close(gWo.cpu().numpy().reshape(H, C), dWo_ref, 5e-3, "Wo grad")
    close(dh16.float().cpu().numpy(), dh_ref, 5e-3, "S dh16")


@pytest.mark.parametrize("n,C", [(300, 16), (9000, 16), (2049, 32)])
def test_fused_readout_f16_evolve_matches_fp64(n, C):
    """dgc_readout_f16_evolve (EvolveGCN-O readout on H2 = relu(.)): dZ2 = dh *
    (H2 > 0) as fp32 and its column sums (the b2 gradient) vs fp64 on the same
    fp16 operands; loss, bo and Wo gradients as the LSTM variant."""
    from paper_2309_03523_b200 import ops
    H, e = 128, 13
    S = 2.0 ** e
    rng = np.random.default_rng(2 * n + C)
    h16 = np.maximum(rng.standard_normal((n, H)), 0).astype(np.float16)  # relu output
    Wo16 = (rng.standard_normal((H, C)) / np.sqrt(H)).astype(np.float16)
    bo = (0.1 * rng.standard_normal(C)).astype(np.float32)
    y = rng.integers(0, C, size=n).astype(np.int32)
    y[rng.random(n) < 0.1] = -1
    scale = 1.0 / n
    tiles, grid = 4 * ((n + 127) // 128), ops.readout_f16_grid(n)
    dz2 = torch.zeros((n, H), device=dev)
    b2p = torch.zeros(tiles * H, device=dev)
    lp = torch.zeros(tiles, device=dev, dtype=torch.float64)
    dp = torch.zeros(tiles * C, device=dev)
    wp = torch.zeros(grid * H * C, device=dev)
    ops.readout_f16_evolve(torch.as_tensor(h16).to(dev), torch.as_tensor(Wo16).to(dev), t(bo),
                           t(y, torch.int32), C, scale, S, dz2, b2p, lp, dp, wp)
    gWo, gbo, gb2 = torch.zeros(H * C, device=dev), torch.zeros(C, device=dev), torch.zeros(H, device=dev)
    ops.reduce_rows_batched([(dp, tiles, C, gbo), (wp, grid, H * C, gWo), (b2p, tiles, H, gb2)])
    torch.cuda.synchronize()
    hd, Wd = h16.astype(np.float64), Wo16.astype(np.float64)
    z = hd @ Wd + bo.astype(np.float64)
    z -= z.max(1, keepdims=True)
    p = np.exp(z) / np.exp(z).sum(1, keepdims=True)
    real = y >= 0
    loss = -np.log(p[np.arange(n)[real], y[real]]).sum()
    dl = p.copy()
    dl[np.arange(n)[real], y[real]] -= 1.0
    dl[~real] = 0.0
    dl *= scale
    dl16 = (dl * S).astype(np.float16).astype(np.float64)
    dz_ref = (dl16 @ Wd.T / S) * (hd > 0)
    assert abs(lp.sum().item() - loss) <= 1e-5 * abs(loss)
    close(gbo.cpu().numpy(), dl.sum(0), 1e-4, "bo grad")
    close(gWo.cpu().numpy().reshape(H, C), hd.T @ dl16 / S, 5e-3, "Wo grad")
    close(dz2.cpu().numpy(), dz_ref, 5e-3, "dZ2")
    close(gb2.cpu().numpy(), dz_ref.sum(0), 5e-3, "b2 grad")


def test_tf32x24_input_pipeline_is_bit_exact():
    """Host pack (round-to-nearest-away to TF32, keep 3 bytes) + device unpack
    equals the device's cvt.rna.tf32 rounding of the fp32 values, bit for bit,
    including ties, carries into the exponent, subnormals, zeros and infinities."""
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(7)
    x = rng.standard_normal(1 << 16).astype(np.float32)
    special = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, 1e-40, -1e-40, 3.4e38, -3.4e38],
                       np.float32)
    ties = (np.arange(1, 1 + 64, dtype=np.uint32) << 13 | 0x1000).view(np.float32)  # exact halves
    near = (np.uint32(0x3FFFF000) + np.arange(64, dtype=np.uint32)).view(np.float32)  # carry into exp
    x = np.concatenate([x, special, ties, -ties, near, np.zeros(2, np.float32)])
    x = x[: len(x) // 4 * 4]
    ref = torch.empty(len(x), device=dev)
    ops.round_tf32(t(x), ref)
    out = torch.empty(len(x), device=dev)
    ops.unpack_tf32x24(torch.as_tensor(ops.pack_tf32x24(x)).to(dev), out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.cpu().numpy().view(np.uint32))


def test_f16_input_pipeline_is_bit_exact():
    """Host fp16 conversion (numpy, round to nearest even) + device unpack equals
    the device's dgc_round_f16 of the fp32 values, bit for bit, including ties,
    fp16 subnormals, zeros, the largest finite values and infinities."""
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(8)
    x = rng.standard_normal(1 << 16).astype(np.float32)
    special = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, 6e-8, -3e-6, 65504.0, -65519.0,
                        1e-40, 2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -25], np.float32)
    ties = (1.0 + (2 * np.arange(1, 65) + 1) * 2.0 ** -11).astype(np.float32)  # exact halves
    x = np.concatenate([x, special, ties, -ties])
    x = x[: len(x) // 8 * 8]
    ref = torch.empty(len(x), device=dev)
    ops.round_f16(t(x), ref)
    out = torch.empty(len(x), device=dev)
    ops.unpack_f16(torch.as_tensor(x.astype(np.float16)).to(dev), out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.cpu().numpy().view(np.uint32))


def test_reduce_rows_batched_equals_separate_calls():
    """The batched bias-gradient reduction is bitwise the per-job dgc_reduce_rows."""
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(11)
    shapes = [(782, 16), (6252, 128), (144, 512), (1, 64), (300, 33)]
    ins = [t(rng.standard_normal((r, w)).astype(np.float32)) for r, w in shapes]
    sep = [torch.zeros(w, device=dev) for _, w in shapes]
    bat = [torch.zeros(w, device=dev) for _, w in shapes]
    for x, (r, w), o in zip(ins, shapes, sep):
        ops.reduce_rows(x, r, w, o)
    ops.reduce_rows_batched([(x, r, w, o) for x, (r, w), o in zip(ins, shapes, bat)])
    torch.cuda.synchronize()
    for a, b in zip(sep, bat):
        assert np.array_equal(a.cpu().numpy(), b.cpu().numpy())


def test_softmax_xent_f16_output_and_step_tail():
    """dgc_softmax_xent_f16: the same loss partials and fp32 dlogits as
    dgc_softmax_xent, plus fp16(scale16 * dlogits) (round to nearest even) and
    the same dlogits column sums; dgc_epoch_finish: fixed-order fp64 loss sum and
    the device step count; dgc_adam_dev_mirror: bitwise the adam + round_tf32 +
    to_f16 sequence it replaces."""
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(11)
    n, C = 5003, 16
    logits = t(rng.standard_normal((n, C)).astype(np.float32) * 3)
    y = rng.integers(0, C, n).astype(np.int32)
    y[::97] = -1  # padding rows
    yt = t(y, torch.int32)
    nb = (n + 255) // 256
    dl, lp, dp = torch.zeros((n, C), device=dev), torch.zeros(nb, dtype=torch.float64, device=dev), \
        torch.zeros(nb * C, device=dev)
    ops.softmax_xent(logits, yt, C, 1.0 / n, dl, lp, dl_partial=dp)
    dl2, lp2, dp2 = torch.zeros_like(dl), torch.zeros_like(lp), torch.zeros_like(dp)
    d16 = torch.zeros((n, C), dtype=torch.float16, device=dev)
    S = 2.0 ** 12
    ops.softmax_xent(logits, yt, C, 1.0 / n, dl2, lp2, dl_partial=dp2, dlogits16=d16, scale16=S)
    d16b = torch.zeros_like(d16)
    ops.softmax_xent(logits, yt, C, 1.0 / n, None, lp2, dl_partial=dp2, dlogits16=d16b, scale16=S)
    torch.cuda.synchronize()
    assert torch.equal(dl2, dl) and torch.equal(lp2, lp) and torch.equal(dp2, dp)
    assert torch.equal(d16, (dl * S).half()) and torch.equal(d16b, d16)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    step = torch.full((1,), 6, dtype=torch.int32, device=dev)
    ops.epoch_finish(lp, loss, step)
    ops.epoch_finish(lp, loss, None)
    torch.cuda.synchronize()
    assert float(loss) == pytest.approx(float(lp.sum()), rel=1e-15) and int(step) == 7
    m = 70001
    p = t(rng.standard_normal(m).astype(np.float32))
    g = t(rng.standard_normal(m).astype(np.float32) * 1e-3)
    mv = [torch.zeros(m, device=dev) for _ in range(4)]
    p2 = p.clone()
    ops.adam(p, g, mv[0], mv[1], 1e-3, 0.9, 0.999, 1e-8, step)
    pr, p16 = torch.zeros_like(p), torch.zeros(m, dtype=torch.float16, device=dev)
    ops.round_tf32(p, pr)
    ops.to_f16(pr, p16)
    pr2, p162 = torch.zeros_like(p), torch.zeros_like(p16)
    ops.adam_mirror(p2, g, mv[2], mv[3], 1e-3, 0.9, 0.999, 1e-8, step, p_r=pr2, p16=p162)
    torch.cuda.synchronize()
    for a, b in ((p2, p), (mv[2], mv[0]), (mv[3], mv[1]), (pr2, pr), (p162, p16)):
        assert torch.equal(a, b)


def test_gemm_cta_cap_same_result():
    """dgc_gemm_max_ctas: a capped grid (the concurrent-GEMM mode) gives bitwise
    the same output and split-K partial reduction as the full grid."""
    from paper_2309_03523_b200 import ops
    rng = np.random.default_rng(12)
    M, N, K = 3000, 128, 512
    A = t(rng.standard_normal((M, K)).astype(np.float32)).half()
    B = t(rng.standard_normal((N, K)).astype(np.float32)).half()
    outs = []
    for cap in (0, 37):
        prev = ops.gemm_max_ctas(cap)
        C = torch.zeros((M, N), device=dev)
        ops.gemm_f16(A, B, C, M, N, K, b_mn=False, ldb=K)
        G = torch.zeros((K, N), device=dev)
        part = torch.zeros(ops.gemm_splits(M, 2, 64) * K * N, device=dev)
        ops.gemm_f16(A, C.half(), G, K, N, M, a_mn=True, lda=K, k_splits=64, partial=part)
        ops.gemm_max_ctas(prev)
        torch.cuda.synchronize()
        outs.append((C.clone(), G.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    ref = A.float() @ B.float().t()
    close(outs[0][0].cpu().numpy(), ref.cpu().numpy(), 2e-3, "capped gemm")
