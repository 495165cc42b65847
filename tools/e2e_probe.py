"""Where the e2e step (bench.py's end-to-end loop) spends time beyond the
device epoch: epochs with / without the next epoch's H2D staging, and the
staging alone."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2309_03523_b200 import DGNNConfig, load_plan_npz
from paper_2309_03523_b200.trainer import DGNNTrainer
from paper_2309_03523_b200.model import synthetic_inputs
pa = load_plan_npz("artifacts/c2/plan.npz")
cfg = DGNNConfig.for_profile(pa.profile, F=128, H=128, C=16, precision="tf32", optimizer="adam", lr=1e-3)
X, y = synthetic_inputs(pa.n_instances, cfg.F, cfg.C, 0)
tr = DGNNTrainer(pa, cfg, None, seed=0, features=X, labels=y, cuda_graph=True)
for _ in range(3): tr.run_epoch()
xs, ys = tr.host_inputs(X, y)
tr.stage_inputs(xs, ys)
def timed(fn, k=10):
    out = []
    for _ in range(k):
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); c0 = time.perf_counter(); r = fn(); c1 = time.perf_counter(); e.record()
        torch.cuda.synchronize()
        out.append((s.elapsed_time(e), (c1 - c0) * 1e3, getattr(r, "wall_ms", 0.0)))
    return np.median(np.array(out), axis=0)
for _ in range(3): tr.run_epoch(next_inputs=(xs, ys))
print("epoch + next H2D staging (e2e loop): event ms, host ms, graph ms", timed(lambda: tr.run_epoch(next_inputs=(xs, ys))))
print("epoch alone:                         ", timed(lambda: tr.run_epoch()))
print("staging alone:                       ", timed(lambda: tr.stage_inputs(xs, ys)))
