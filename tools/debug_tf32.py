import os, sys
sys.path.insert(0, ".")
import numpy as np
from pathlib import Path
from tests.test_gpu_trainer import run_pair
from paper_2309_03523_b200 import load_plan_npz
pa = load_plan_npz(Path("artifacts/t4/plan.npz"))
for tc in ("0", "1"):
    os.environ["DGC_TC_RNN"] = tc
    out, tr, orc = run_pair(pa, dict(F=32, H=64, C=16, rnn="lstm", n_rnn=2), "off", epochs=1, precision="tf32")
    rep, o, grads = out[0]
    print("TC_RNN", tc, "loss rel", abs(rep.loss - o["loss"]) / o["loss"])
    for k, g in grads.items():
        ref = o["grads"][k]
        print("   ", k, f"{np.abs(g - ref).max() / np.abs(ref).max():.2e}", f"rel-norm {np.linalg.norm(g-ref)/np.linalg.norm(ref):.2e}")
