import sys
sys.path.insert(0, ".")
import torch
from paper_2309_03523_b200 import ops
M, N, K = (int(x) for x in sys.argv[1:4])
a_mn, b_mn = int(sys.argv[4]), int(sys.argv[5])
prec = int(sys.argv[6]) if len(sys.argv) > 6 else 1
A = torch.randn((K, M) if a_mn else (M, K), device="cuda")
B = torch.randn((K, N) if b_mn else (N, K), device="cuda")
C = torch.zeros((M, N), device="cuda")
f = lambda: ops.gemm(A, B, C, M, N, K, a_mn=bool(a_mn), b_mn=bool(b_mn), precision=prec)
f(); torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): f()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
nb = 4 * (M * K + K * N + M * N)
print(f"gemm {M}x{N}x{K} a_mn={a_mn} b_mn={b_mn} p={prec}: {ms*1e3:.1f} us  {nb/ms/1e6:.0f} GB/s")
