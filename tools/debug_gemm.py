import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2309_03523_b200 import ops
rng = np.random.default_rng(5)
n, F, H = 20000, 128, 96
X = rng.standard_normal((n, F)).astype(np.float32)
dY = rng.standard_normal((n, H)).astype(np.float32)
ref = X.astype(np.float64).T @ dY.astype(np.float64)
# fp32 sequential-ish reference error scale (numpy fp32 matmul)
r32 = X.T @ dY
print("numpy fp32 err", np.abs(r32 - ref).max() / np.abs(ref).max())
Xd, Yd = torch.tensor(X, device="cuda"), torch.tensor(dY, device="cuda")
part = torch.zeros(700 * F * H, device="cuda")
for prec in (1, 3):
    for ks in (1, 5, 20, 79, 157, 625):
        C = torch.zeros((F, H), device="cuda")
        ops.gemm(Xd, Yd, C, F, H, n, a_mn=True, precision=prec, k_splits=ks, partial=part)
        torch.cuda.synchronize()
        d = C.cpu().numpy() - ref
        err = np.abs(d).max() / np.abs(ref).max()
        bias = (d * np.sign(ref)).mean() / np.abs(ref).mean()
        print("prec", prec, "ksplit", ks, f"err {err:.3e} signed-bias {bias:.3e}")
