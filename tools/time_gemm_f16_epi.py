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
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def t(fn, k=20):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    return sorted(ts)[k // 2]
for rep in range(1):
    print("relu only   :", round(t(lambda: ops.gemm_f16(A, W, None, M, N, K, act=1, C16=C16)), 1))
    print("no bias     :", round(t(lambda: ops.gemm_f16(A, W, None, M, N, K, C16=C16)), 1))
    print("bias+relu   :", round(t(lambda: ops.gemm_f16(A, W, None, M, N, K, bias=b, act=1, C16=C16)), 1))
    print("bias        :", round(t(lambda: ops.gemm_f16(A, W, None, M, N, K, bias=b, C16=C16)), 1))
# the backward's masked GEMM: dZ1 = (dY2 W2^T) * (H1 > 0) as fp16, + bias-gradient column sums
R16 = torch.randn((M, N), device=dev).half()
cs = torch.zeros(4 * ((M + 127) // 128) * N, device=dev)
print("relu16      :", round(t(lambda: ops.gemm_f16(A, W, None, M, N, K, relu16=R16, C16=C16)), 1))
print("colsum      :", round(t(lambda: ops.gemm_f16(A, W, None, M, N, K, colsum_partial=cs, C16=C16)), 1))
print("relu16+csum :", round(t(lambda: ops.gemm_f16(A, W, None, M, N, K, relu16=R16, colsum_partial=cs, C16=C16)), 1))
