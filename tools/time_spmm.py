"""SpMM variants on the C2 CSR: fp32 vs bf16 gathered operand, unroll depth
(DGC_SPMM_UNR), with CUDA events; prints us per launch and algorithmic GB/s."""
import os
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2309_03523_b200 import load_plan_npz, _native
from paper_2309_03523_b200.layout import build_layout

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
pa = load_plan_npz(f"artifacts/{cfg}/plan.npz") if os.path.exists(f"artifacts/{cfg}/plan.npz") else None
if pa is None:
    from paper_2309_03523_b200 import single_device
    pa = single_device(load_plan_npz(f"artifacts/{cfg}d8/plan.npz"))
L = build_layout(pa, 0)
dev = "cuda"
rp = torch.tensor(np.asarray(L.row_ptr, np.int32), device=dev); col = torch.tensor(np.asarray(L.col, np.int32), device=dev)
n = rp.numel() - 1; nnz = col.numel()
deg = np.diff(np.asarray(L.row_ptr)).astype(np.float64)
dinv = torch.tensor(1.0 / np.sqrt(deg), dtype=torch.float32, device=dev)
W = int(sys.argv[2]) if len(sys.argv) > 2 else 128
g = torch.Generator(device=dev).manual_seed(0)
Y = torch.randn((n, W), device=dev, generator=g)
Yb = Y.to(torch.bfloat16)
out = torch.empty((n, W), device=dev)
ref = torch.empty((n, W), device=dev)
lib = _native.lib()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
p = lambda t: t.data_ptr()
def run(Yt, dt, o):
    _native.check(lib.dgc_spmm_csr_ex(p(rp), p(col), p(dinv), p(Yt), dt, None, p(o), None, n, 0, W, 0, None), "spmm")
run(Y, 0, ref)
yb_as_f = Yb.float()
ref_b = torch.empty_like(ref); run(yb_as_f, 0, ref_b)
for unr in (2, 4, 8):
    os.environ["DGC_SPMM_UNR"] = str(unr)
    for name, Yt, dt, eb in (("fp32", Y, 0, 4), ("bf16", Yb, 1, 2)):
        run(Yt, dt, out); torch.cuda.synchronize()
        if dt == 1:
            err = float((out - ref_b).abs().max() / ref_b.abs().max())
        else:
            err = float((out - ref).abs().max())
        ts = []
        for _ in range(5):
            flush.zero_()
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(); run(Yt, dt, out); e.record(); torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        t = float(np.median(ts))
        alg = eb * W * n + 4 * W * n + 4 * (n + 1) + 4 * nnz + 4 * n
        print(f"{cfg} W={W} unr={unr} {name}: {t:7.1f} us  alg {alg/t/1e3:7.0f} GB/s  gather {nnz*W*eb/t/1e3:7.0f} GB/s  err {err:.1e}")
