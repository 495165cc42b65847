"""Host-side logic of the input pipeline and the K-segmented GEMM work split
(CPU; the device halves are in tests/test_gpu_kernels.py / test_gpu_trainer.py)."""
import numpy as np

from paper_2309_03523_b200 import ops
from paper_2309_03523_b200.trainer import k_segment_items


def _rna_tf32_reference(x):
    """Round to nearest TF32, ties away from zero, by explicit arithmetic on the
    magnitude (independent of the bit trick in ops.pack_tf32x24)."""
    out = np.empty_like(x)
    for i, v in enumerate(x.astype(np.float64)):
        if not np.isfinite(v) or v == 0.0:
            out[i] = v
            continue
        m, e = np.frexp(abs(v))             # |v| = m 2^e, m in [0.5, 1)
        e = max(e, -125)                    # fp32 subnormals: fixed quantum
        q = 2.0 ** (e - 11)                 # TF32 keeps 11 significant bits
        r = np.floor(abs(v) / q + 0.5) * q  # ties away (magnitude rounding)
        out[i] = np.float32(np.copysign(r, v))
    return out


def test_pack_tf32x24_matches_round_to_nearest_away():
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.standard_normal(4000).astype(np.float32) * 10.0 ** rng.integers(-20, 20, 4000),
                        (np.arange(1, 65, dtype=np.uint32) << 13 | 0x1000).view(np.float32),  # ties
                        np.array([0.0, -0.0, 1.0, -2.5, 3.0e38, -1e-30], np.float32)]).astype(np.float32)
    x = x[: len(x) // 4 * 4]
    packed = ops.pack_tf32x24(x)
    assert packed.dtype == np.uint8 and packed.size == 3 * x.size
    # host-side expansion (the device kernel does the same shift)
    b = packed.reshape(-1, 3).astype(np.uint32)
    u = (b[:, 0] << 8) | (b[:, 1] << 16) | (b[:, 2] << 24)
    got = u.view(np.float32)
    ref = _rna_tf32_reference(x)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_k_segment_items_cover_every_k_block_in_two_waves():
    rng = np.random.default_rng(0)
    for T in (8, 64, 128):
        sizes = (rng.integers(0, 3000, T) // 32) * 32
        sizes[rng.integers(0, T)] = 0          # an empty snapshot
        seg = np.concatenate([[0], np.cumsum(sizes)])
        for fp32 in (False, True):
            items, ptr = k_segment_items(seg, T, fp32)
            assert len(ptr) == T + 1 and ptr[-1] == len(items)
            for t in range(T):                  # each snapshot's items tile its k-blocks in order
                kb = seg[t] // 32
                for a, nk in items[ptr[t]:ptr[t + 1]]:
                    assert a == kb and nk >= 1
                    kb += nk
                assert kb == seg[t + 1] // 32
            if fp32:
                assert max(nk for _, nk in items) <= 16
            elif seg[T] // 32 >= 296:
                assert len(items) <= 296        # at most two waves of 148
                assert len(items) >= 296 - T    # and nearly full
