"""K1 SpMM variants (DGC_SPMM_STREAM / DGC_SPMM_MODE, read once per process) on a plan's CSR:
fp16-row (dgc_spmm_csr_h) and fp32-row (dgc_spmm_csr) launches, CUDA events,
L2 flushed per launch; prints us per launch and a hash of the output (the
variants must agree bitwise). usage: python tools/time_spmm_modes.py c2|c3 [W]"""
import hashlib
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
g = torch.Generator(device=dev).manual_seed(0)
Y = torch.randn((n, W), device=dev, generator=g)
Y16 = Y.half()
out = torch.empty((n, W), device=dev)
o16 = torch.empty((n, W), device=dev, dtype=torch.float16)
bias = torch.randn(W, device=dev, generator=g)
work = torch.zeros(2, dtype=torch.int32, device=dev)
lib = _native.lib()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def t_of(run):
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); run(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return float(np.median(ts))


def h(*ts):
    m = hashlib.sha1()
    for t in ts:
        m.update(t.cpu().numpy().tobytes())
    return m.hexdigest()[:12]


mode = os.environ.get("DGC_SPMM_STREAM", os.environ.get("DGC_SPMM_MODE", os.environ.get("DGC_SPMM_LD", "-")))
runh = lambda: _native.check(lib.dgc_spmm_csr_h(rp.data_ptr(), col.data_ptr(), dinv.data_ptr(),
                                                Y16.data_ptr(), bias.data_ptr(), None, o16.data_ptr(),
                                                1.0, n, W, 1, work.data_ptr(), None), "spmm_h")
t = t_of(runh)
print(f"{cfg} mode {mode:>3} fp16 rows W={W} n={n} nnz={nnz}: {t:7.1f} us  "
      f"{nnz / t / 1e3:6.2f} G nbr rows/s  hash {h(o16)}")
runf = lambda: _native.check(lib.dgc_spmm_csr_x(rp.data_ptr(), col.data_ptr(), dinv.data_ptr(),
                                                Y.data_ptr(), bias.data_ptr(), out.data_ptr(), None,
                                                None, n, 0, W, 1, work.data_ptr(), 1.0, None), "spmm_x")
t = t_of(runf)
alg = 8 * W * n + 4 * (n + 1) + 4 * nnz + 4 * n
print(f"{cfg} mode {mode:>3} fp32 rows W={W}: {t:7.1f} us  alg {alg / t / 1e3:6.0f} GB/s  "
      f"{nnz / t / 1e3:6.2f} G nbr rows/s  hash {h(out)}")
