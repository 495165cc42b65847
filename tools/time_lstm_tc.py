import sys, time
# per-position timestamps need a build with them compiled in: make clean && make DGC_TS=1
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2309_03523_b200 import ops
from paper_2309_03523_b200.layout import pack_sequences_native
H = int(sys.argv[1]) if len(sys.argv) > 1 else 128
rng = np.random.default_rng(0)
lengths = np.full(6250, 32)
seq, pos, mask, _ = pack_sequences_native(lengths)
R, L = seq.shape
offs = np.concatenate([[0], np.cumsum(lengths)])
n = int(offs[-1])
slot_row = np.where(seq >= 0, offs[np.maximum(seq, 0)] + pos, -1).astype(np.int32).reshape(-1)
dev = "cuda"
gx = torch.randn((n, 4 * H), device=dev)
Ut = torch.randn((4 * H, H), device=dev) / H ** 0.5
U = Ut.t().contiguous()
sr = torch.tensor(slot_row, device=dev)
sm = torch.tensor(mask.reshape(-1), device=dev)
sc = torch.full((R * L,), -1, dtype=torch.int32, device=dev)
carry = torch.zeros((1, 2 * H), device=dev)
hc = torch.zeros((n, 2 * H), device=dev)
save = torch.zeros((n, 7 * H), device=dev)
for name, fn in (("tc", lambda: ops.rnn_fwd_tc(1, gx, Ut, sr, sm, sc, carry, R, L, H, 2 * H, hc, hc[:, H:], save)),
                 ("simt", lambda: ops.rnn_fwd(1, gx, U, sr, sm, sc, carry, R, L, H, 2 * H, hc, hc[:, H:], save))):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3): fn()
    e.record(); torch.cuda.synchronize()
    print(name, "H", H, "R", R, "L", L, f"{s.elapsed_time(e)/3:.3f} ms")
import ctypes
from paper_2309_03523_b200 import _native
lib = _native.lib()
ops.rnn_fwd_tc(1, gx, Ut, sr, sm, sc, carry, R, L, H, 2 * H, hc, hc[:, H:], save); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (256 * 8))()
lib.dgc_debug_lstm_timestamps(buf, 256 * 8)
ts = np.array(buf[:L * 3], dtype=np.float64).reshape(L, 3)
t0 = ts[0, 0]
for p in range(min(L, 6)):
    print(f"p={p} mma_start {(ts[p,0]-t0)/1e3:8.2f} acc_ready {(ts[p,1]-t0)/1e3:8.2f} epi_done {(ts[p,2]-t0)/1e3:8.2f} us")
d = np.diff(ts[:, 0])
print("per-step us: mma", np.mean(ts[:, 1] - ts[:, 0]) / 1e3, "epi", np.mean(ts[:, 2] - ts[:, 1]) / 1e3, "step", np.mean(d) / 1e3)
