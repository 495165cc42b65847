"""Per-position timeline of the LSTM BPTT cluster kernel at the C2 bench
workload (the last LSTM launch of an eager epoch = layer-1 BPTT), from the
globaltimer stamps of CTA 0. Needs a build with them: make clean && make DGC_TS=1"""
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
buf = (ctypes.c_ulonglong * (256 * 8))()
_native.lib().dgc_debug_lstm_timestamps(buf, 256 * 8)
L = pa.T
ts = np.array(buf[:L * 8], dtype=np.float64).reshape(L, 8)
t0 = ts[0, 0]
print("BPTT per position (us from its start): acc_ready, tmem+send done, recv done, lc0 done, lc1 done")
for t in range(L):
    r = ts[t]
    print(f"t={t:2d} start {(r[0]-t0)/1e3:8.2f} | " + " ".join(f"{(r[k]-r[0])/1e3:6.2f}" for k in (1, 3, 4, 5, 2)))
d = ts[1:]
ph = lambda a, b: np.mean(d[:, b] - d[:, a]) / 1e3
print(f"mean per position (us): wait-acc {ph(0,1):.2f} tmem+send {ph(1,3):.2f} recv-wait {ph(3,4):.2f} "
      f"lc0 {ph(4,5):.2f} lc1 {ph(5,2):.2f} epi_done->next {np.mean(ts[1:, 0] - ts[:-1, 2]) / 1e3:.2f} "
      f"position {np.mean(np.diff(ts[:, 0])) / 1e3:.2f}")
wb = (ctypes.c_ulonglong * (256 * 32))()
_native.lib().dgc_debug_lstm_timestamps_warps(wb, 256 * 32)
w = np.array(wb[:L * 32], dtype=np.float64).reshape(L, 32)[:, :12]
rel = (w[1:] - ts[1:, 0:1]) / 1e3  # per epilogue warp: chunk-1 done, us after the position start
print("per-warp chunk-1 done (us after position start, mean over positions):", np.round(rel.mean(0), 2))
print("slowest warp minus warp 0, mean:", round(float((rel.max(1) - rel[:, 0]).mean()), 2))
# MMA warp: last k-block's a_full seen for position t (stamp 7) vs the epilogue's acc ready at t+1 (stamp 1)
mm = ts[:-1, 7]
print("MMA sees the last da k-block -> epilogue sees acc (next position), us:", round(float(np.mean(ts[1:, 1] - mm) / 1e3), 2),
      "; last warp's chunk-1 done -> MMA sees it, us:", round(float(np.mean(mm - w[:-1].max(1)) / 1e3), 2))
