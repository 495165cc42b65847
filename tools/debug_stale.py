import sys
sys.path.insert(0, ".")
import numpy as np
from pathlib import Path
from tests.test_gpu_trainer import run_pair
from paper_2309_03523_b200 import load_plan_npz

pa = load_plan_npz(Path("artifacts/t2/plan.npz"))
out, tr, orc = run_pair(pa, dict(F=16, H=16, C=16, rnn="gru", n_rnn=1), "relax", epochs=2)
for rep, o, grads in out:
    print("epoch", rep.epoch, "loss", rep.loss, o["loss"], "theta", rep.stale_detail, o["theta"], o["d_r"])
    for k, g in grads.items():
        ref = o["grads"][k]
        print("  ", k, np.abs(g - ref).max() / np.abs(ref).max())
for d, sh in enumerate(tr.shards):
    for l in range(2):
        got = sh.scache[l].send.cpu().numpy().astype(bool)
        ref = out[-1][1]["send"][f"s{l}"][d]
        print("shard", d, "layer", l, "send mism", int((got != ref).sum()), "sent", int(got.sum()), len(got))
        halo = sh.Yext[l][sh.n:].cpu().numpy()
        print("   halo diff", np.abs(halo - orc.halo[l][d]).max())
    tsend = sh.tcache[0].send.cpu().numpy().astype(bool)
    print("   tsend mism", int((tsend != out[-1][1]["send"]["t0"][d]).sum()))
    print("   carry diff", np.abs(sh.carry[0][:sh.lay.n_carry].cpu().numpy() - orc.carry[0][d]).max() if sh.lay.n_carry else 0)
