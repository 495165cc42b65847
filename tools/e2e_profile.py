import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
from paper_2309_03523_b200 import DGNNConfig
from paper_2309_03523_b200.trainer import DGNNTrainer
from paper_2309_03523_b200.model import init_params, synthetic_inputs
from pathlib import Path
from paper_2309_03523_b200 import load_plan_npz
pa = load_plan_npz(Path("artifacts/c2/plan.npz"))
cfg = DGNNConfig(F=128, H=128, C=16, rnn="lstm", n_rnn=2, optimizer="adam", lr=1e-3, precision="tf32")
X, y = synthetic_inputs(pa.n_instances, cfg.F, cfg.C, 0)
tr = DGNNTrainer(pa, cfg, None, features=X, labels=y, params=init_params(cfg, 0), cuda_graph=True)
for _ in range(3): tr.run_epoch()
xs, ys = tr.host_inputs(X, y)
tr.stage_inputs(xs, ys)
import cProfile, pstats
ts = []
for i in range(15):
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); c0 = time.perf_counter()
    rep = tr.run_epoch(next_inputs=(xs, ys)); l = float(rep.loss)
    c1 = time.perf_counter(); e.record(); torch.cuda.synchronize()
    ts.append((s.elapsed_time(e), (c1 - c0) * 1e3, rep.wall_ms))
print("e2e ms, cpu ms, graph ms:", np.median(np.array(ts), axis=0))
pr = cProfile.Profile(); pr.enable()
for i in range(10): rep = tr.run_epoch(next_inputs=(xs, ys))
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
