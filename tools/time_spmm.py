"""K1 SpMM on a plan's CSR (CUDA events, L2 flushed per launch): us per launch,
algorithmic GB/s and the gathered-row rate. usage: python tools/time_spmm.py [c2|c3|c5] [W]
(the bf16-operand and TMA-staged variants measured in round 2 were built at
commit 6261801 / the r2 session; numbers in profiles/r2_summary.md)"""
import os
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2309_03523_b200 import load_plan_npz, single_device, _native
from paper_2309_03523_b200.layout import build_layout

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 128
pa = (load_plan_npz(f"artifacts/{cfg}/plan.npz") if os.path.exists(f"artifacts/{cfg}/plan.npz")
      else single_device(load_plan_npz(f"artifacts/{cfg}d8/plan.npz")))
L = build_layout(pa, 0)
dev = "cuda"
rp = torch.tensor(np.asarray(L.row_ptr, np.int32), device=dev)
col = torch.tensor(np.asarray(L.col, np.int32), device=dev)
n = rp.numel() - 1
nnz = col.numel()
deg = np.diff(np.asarray(L.row_ptr)).astype(np.float64)
dinv = torch.tensor(1.0 / np.sqrt(deg), dtype=torch.float32, device=dev)
Y = torch.randn((n, W), device=dev, generator=torch.Generator(device=dev).manual_seed(0))
out = torch.empty((n, W), device=dev)
lib = _native.lib()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
run = lambda: _native.check(lib.dgc_spmm_csr(rp.data_ptr(), col.data_ptr(), dinv.data_ptr(),
                                             Y.data_ptr(), None, out.data_ptr(), n, W, 0, None), "spmm")
run()
ts = []
for _ in range(5):
    flush.zero_()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); run(); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e) * 1e3)
t = float(np.median(ts))
alg = 8 * W * n + 4 * (n + 1) + 4 * nnz + 4 * n
print(f"{cfg} W={W} rows {n} nnz {nnz}: {t:7.1f} us  alg {alg / t / 1e3:7.0f} GB/s  "
      f"gathered rows {nnz * W * 4 / t / 1e3:7.0f} GB/s")
work = torch.zeros(2, dtype=torch.int32, device=dev)
out3 = torch.empty_like(out)
rund = lambda: _native.check(lib.dgc_spmm_csr_x(rp.data_ptr(), col.data_ptr(), dinv.data_ptr(),
                                                Y.data_ptr(), None, out3.data_ptr(), None, None, n,
                                                0, W, 0, work.data_ptr(), None), "spmm_x")
rund(); torch.cuda.synchronize()
assert torch.equal(out3, out)
ts = []
for _ in range(5):
    flush.zero_()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); rund(); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e) * 1e3)
t = float(np.median(ts))
print(f"{cfg} W={W} dynamic rows: {t:7.1f} us  alg {alg / t / 1e3:7.0f} GB/s  "
      f"gathered rows {nnz * W * 4 / t / 1e3:7.0f} GB/s")
