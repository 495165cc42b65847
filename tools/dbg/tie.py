import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np
from pathlib import Path
import test_gpu_trainer as T
from paper_2309_03523_b200 import load_plan_npz
pa = load_plan_npz(Path('/root/repo/artifacts/t4/plan.npz'))
out, tr, orc = T.run_pair(pa, dict(F=16, H=16, C=16, rnn="lstm", n_rnn=2), "relax", epochs=4, fraction=0.3)
for e in orc.tie_log[:40]:
    print(e['epoch'], e['cache'], e['device'], e['key'], 'dist', e['dist'], 'theta', e['theta'], 'rel', (e['dist']-e['theta'])/e['theta'], 'scale', e['scale'])
for rep,o,_ in out:
    print(rep.epoch, rep.stale_detail, o['theta'], o['d_r'])
