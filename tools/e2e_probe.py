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
def pipelined(k, stage=True):
    prev = None
    for _ in range(k):
        p = tr.submit_epoch(next_inputs=(xs, ys) if stage else None)
        if prev is not None:
            float(prev.result().loss)
        prev = p
    float(prev.result().loss)
    torch.cuda.synchronize()
for stage in (True, False):
    pipelined(3, stage)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); c0 = time.perf_counter(); pipelined(10, stage); c1 = time.perf_counter(); e.record(); torch.cuda.synchronize()
    print(f"pipelined x10 stage={stage}: {s.elapsed_time(e) / 10:.3f} ms/step (host {(c1 - c0) * 100:.3f} ms/step)")
# graph epochs back to back without any host read
g, _ = next(iter(tr._graphs.values()))
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): g.replay()
e.record(); torch.cuda.synchronize()
print(f"raw graph replay x10: {s.elapsed_time(e) / 10:.3f} ms/step")
slot = torch.empty(1, dtype=torch.float64, pin_memory=True)
src = torch.zeros(1, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
s.record()
for _ in range(10):
    g.replay(); slot.copy_(src, non_blocking=True)
e.record(); torch.cuda.synchronize()
print(f"graph replay + 8-B D2H copy x10: {s.elapsed_time(e) / 10:.3f} ms/step")
torch.cuda.synchronize()
s.record()
for _ in range(10):
    g.replay(); ev = torch.cuda.Event(); ev.record()
e.record(); torch.cuda.synchronize()
print(f"graph replay + event x10: {s.elapsed_time(e) / 10:.3f} ms/step")
torch.cuda.synchronize()
s.record(); c0 = time.perf_counter()
pend = []
for _ in range(10):
    pend.append(tr.submit_epoch())
    if len(pend) > 1: pend[-2].result()
pend[-1].result()
e.record(); torch.cuda.synchronize()
print(f"submit_epoch x10 (no staging): {s.elapsed_time(e) / 10:.3f} ms/step; host {(time.perf_counter() - c0) * 100:.3f}")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(10):
    tr.submit_epoch().result()
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(8)
