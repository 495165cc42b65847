"""The C2 LSTM input-gradient GEMM shape in isolation: dx[200000, 128] =
(S dgx16)[200000, 512] Wx16[128, 512]^T / S (fp16 operands, fp32 out), and the
stacked weight-gradient GEMM [x16; h_in16]^T dgx16 (K = 200000)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2309_03523_b200 import ops
M, N, K = 200000, 128, 512
dev = "cuda"
dgx = (torch.randn((M, K), device=dev) * 0.1).half()
W = (torch.randn((N, K), device=dev) * 0.1).half()
C = torch.empty((M, N), device=dev)
x16 = torch.randn((M, 128), device=dev).half()
save = torch.randn((M, 384), device=dev).half()   # compact save rows (3H fp16 = h_in | c_in | gates)
G = torch.zeros((256, 512), device=dev)
part = torch.zeros((ops.gemm_splits(M, 2, 148) * 256 * 512,), device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def t(fn, k=10):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    return sorted(ts)[k // 2]


dx = lambda: ops.gemm_f16(dgx, W, C, M, N, K, b_mn=False, ldb=K)
dw = lambda: ops.gemm_f16_stacked_a(x16, save, dgx, G, 128, 256, K, M, a_mn=True, lda0=128, lda1=384,
                                    ldb=K, ldc=K, k_splits=148, partial=part)
print(f"dx  [200000x128x512]: {t(dx):.1f} us ({(M * K * 2 + M * N * 4) / t(dx) / 1e3:.0f} GB/s)")
print(f"dW  [256x512x200000] stacked: {t(dw):.1f} us")
if len(sys.argv) > 1 and sys.argv[1] == "once":
    dx(); torch.cuda.synchronize()
