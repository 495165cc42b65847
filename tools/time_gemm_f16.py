"""fp16 GEMM variants at the C2 structure-encoder shape (M = 200000, N = K = 128)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2309_03523_b200 import ops
M, N, K = 200000, 128, 128
dev = "cuda"
A = torch.randn((M, K), device=dev).half()
W = torch.randn((K, N), device=dev).half() * 0.1
b = torch.randn(N, device=dev)
C16 = torch.empty((M, N), device=dev, dtype=torch.float16)
C = torch.empty((M, N), device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def t(fn, k=10):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    return sorted(ts)[k // 2]
print("fp16-only out, no bias     :", t(lambda: ops.gemm_f16(A, W, None, M, N, K, C16=C16)))
print("fp16-only out, bias + relu :", t(lambda: ops.gemm_f16(A, W, None, M, N, K, bias=b, act=1, C16=C16)))
print("fp16-only out, relu only   :", t(lambda: ops.gemm_f16(A, W, None, M, N, K, act=1, C16=C16)))
print("fp16-only out, bias only   :", t(lambda: ops.gemm_f16(A, W, None, M, N, K, bias=b, C16=C16)))
print("fp32 out (TMA), bias+relu  :", t(lambda: ops.gemm_f16(A, W, C, M, N, K, bias=b, act=1)))
Af = A.float(); Wf = W.float()
print("TF32, fp32 out, bias+relu  :", t(lambda: ops.gemm(Af, Wf, C, M, N, K, precision=1, bias=b, act=1)))
