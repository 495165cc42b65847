"""The two largest C2 backward GEMMs in isolation (trainer shapes and strides):
stacked [dWx; dU] = [x; h_in]^T dgx and dh2 = dgx Wx^T; CUDA-event timed with an
L2 flush before each launch. usage: python tools/time_gemm_c2.py [stacked|dh2|both]"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2309_03523_b200 import ops
n, H, G = 200000, 128, 4
GH = G * H
dev = "cuda"
which = sys.argv[1] if len(sys.argv) > 1 else "both"
hbuf = torch.randn((n, 2 * H), device=dev)          # x = h|c of the layer below (ld 2H)
save = torch.randn((n, 7 * H), device=dev)          # h_in = save[:, :H] (ld 7H)
dgx = torch.randn((n, GH), device=dev)
Wx = torch.randn((H, GH), device=dev)
gW = torch.zeros((2 * H, GH), device=dev)
dh2 = torch.zeros((n, H), device=dev)
ks = max(1, min(148, (n // 32) // 4))
part = torch.zeros(ops.gemm_splits(n, 1, ks) * 2 * H * GH, device=dev)
flush = torch.empty(320 * 2 ** 20 // 4, device=dev)
fs = {"stacked": lambda: ops.gemm_stacked_a(hbuf, save, dgx, gW, H, 2 * H, GH, n, a_mn=True,
                                            lda0=2 * H, lda1=7 * H, ldb=GH, ldc=GH, precision=1,
                                            k_splits=ks, partial=part),
      "dh2": lambda: ops.gemm(dgx, Wx, dh2, n, H, GH, b_mn=False, ldb=GH, precision=1)}
for name, f in fs.items():
    if which not in (name, "both"):
        continue
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); f(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    nb = 4 * n * (2 * H + GH) if name == "stacked" else 4 * n * (GH + H)
    print(f"{name}: {ms*1e3:.1f} us, {nb/ms/1e6:.0f} GB/s algorithmic")
