"""Per-position timeline of the 2-SM LSTM BPTT kernel (lstm_bwd_tc2m) at the C2
bench workload, from the globaltimer stamps of CTAs 0 (MMA issuer) and 1.
Needs a build with them: make clean && make DGC_TS=1"""
import ctypes
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2309_03523_b200 import DGNNConfig, load_plan_npz, _native
from paper_2309_03523_b200.trainer import DGNNTrainer

pa = load_plan_npz("artifacts/c2/plan.npz")
cfg = DGNNConfig.for_profile(pa.profile, F=128, H=128, C=16, precision="tf32", optimizer="adam", lr=1e-3)
tr = DGNNTrainer(pa, cfg, None, seed=0)
for _ in range(3):
    tr.run_epoch()
torch.cuda.synchronize()
L = pa.T
buf = (ctypes.c_ulonglong * (256 * 16))()
_native.lib().dgc_debug_lstm_timestamps(buf, 256 * 16)
a = np.array(buf, dtype=np.float64)
ts0 = a[:256 * 8].reshape(256, 8)[:L]
ts1 = a[256 * 8:].reshape(256, 8)[:L]
wb = (ctypes.c_ulonglong * (256 * 32))()
_native.lib().dgc_debug_lstm_timestamps_warps(wb, 256 * 32)
w = np.array(wb, dtype=np.float64).reshape(256, 32)[:L]
T0 = ts0[0, 0]
for name, ts in (("CTA0", ts0), ("CTA1", ts1)):
    d = ts[1:]
    ph = lambda a, b: np.mean(d[:, b] - d[:, a]) / 1e3
    print(f"{name} per position (us): wait-acc {ph(0,1):.2f} tmem {ph(1,3):.2f} lc0 {ph(3,4):.2f} "
          f"lc1 {ph(4,5):.2f} lc2 {ph(5,6):.2f} lc3 {ph(6,2):.2f} position {np.mean(np.diff(ts[:, 0])) / 1e3:.2f}")
for t in range(3, 6):
    print(f"t={t} CTA0 start {(ts0[t,0]-T0)/1e3:.2f} acc {(ts0[t,1]-T0)/1e3:.2f} done {(ts0[t,2]-T0)/1e3:.2f} | "
          f"CTA1 start {(ts1[t,0]-T0)/1e3:.2f} acc {(ts1[t,1]-T0)/1e3:.2f} done {(ts1[t,2]-T0)/1e3:.2f} | "
          f"MMA first kb {(ts1[t,7]-T0)/1e3:.2f} last kb {(ts0[t,7]-T0)/1e3:.2f} | "
          f"last warp done CTA0 {(w[t,:12].max()-T0)/1e3:.2f} CTA1 {(w[t,16:28].max()-T0)/1e3:.2f}")
mm = ts0[:-1, 7]
print("MMA sees last k-block -> CTA0 sees acc (next position), us:", round(float(np.mean(ts0[1:, 1] - mm) / 1e3), 2))
print("last warp (both CTAs) done -> MMA sees last k-block, us:",
      round(float(np.mean(mm - np.maximum(w[:-1, :12].max(1), w[:-1, 16:28].max(1))) / 1e3), 2))
k0 = w[0, 30]
print(f"kernel (CTA0): first position starts {(ts0[0,0]-k0)/1e3:.2f} us after setup, B resident at {(w[0,31]-k0)/1e3:.2f}, "
      f"last position done {(ts0[L-1,2]-k0)/1e3:.2f}, exit {(w[1,30]-k0)/1e3:.2f} us")
