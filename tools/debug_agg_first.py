import os, sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
from pathlib import Path
from test_gpu_trainer import run_pair
from paper_2309_03523_b200 import load_plan_npz, single_device
pa = single_device(load_plan_npz(Path("artifacts") / "t2" / "plan.npz"))
out, tr, _ = run_pair(pa, dict(F=32, H=64, C=16, rnn="lstm", n_rnn=2), "off", epochs=1)
sh = tr.shards[0]
print("agg_first", sh.agg_first)
for rep, o, grads in out:
    for k in ("W1", "b1", "W2", "b2"):
        g, ref = grads[k], o["grads"][k]
        err = np.abs(g - ref)
        i = np.unravel_index(np.argmax(err), err.shape)
        print(k, "max err", err.max() / np.abs(ref).max(), "at", i, g[i], ref[i], "n_bad(>1e-4)", int((err > 1e-4 * np.abs(ref).max()).sum()), "of", err.size)
# H1 near zero?
import torch
H1 = sh.Hl[0].cpu().numpy()
print("H1 exact zeros", int((H1 == 0).sum()), "tiny pos", int(((H1 > 0) & (H1 < 1e-6)).sum()))
