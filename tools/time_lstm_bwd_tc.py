import sys
# per-position timestamps need a build with them compiled in: make clean && make DGC_TS=1
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2309_03523_b200 import ops
from paper_2309_03523_b200.layout import pack_sequences_native
H = int(sys.argv[1]) if len(sys.argv) > 1 else 128
lengths = np.full(6250, 32)
seq, pos, mask, _ = pack_sequences_native(lengths)
R, L = seq.shape
offs = np.concatenate([[0], np.cumsum(lengths)])
n = int(offs[-1])
slot_row = np.where(seq >= 0, offs[np.maximum(seq, 0)] + pos, -1).astype(np.int32).reshape(-1)
dev = "cuda"
U = torch.randn((H, 4 * H), device=dev) / H ** 0.5
sr = torch.tensor(slot_row, device=dev); sm = torch.tensor(mask.reshape(-1), device=dev)
save = torch.rand((n, 7 * H), device=dev); dh = torch.randn((n, H), device=dev)
dgx = torch.zeros((n, 4 * H), device=dev)
tiles = ops.rnn_tc_tiles(R, H)
bp = torch.zeros((tiles, 4 * H), device=dev); scr = torch.zeros(((R + 127) // 128 * 128, H), device=dev)
fn = lambda: ops.rnn_bwd_tc(1, U, sr, sm, R, L, H, save, dh, dgx, scr, bias_partial=bp)
fn(); torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3): fn()
e.record(); torch.cuda.synchronize()
print("lstm bwd tc H", H, f"{s.elapsed_time(e)/3:.3f} ms")
import ctypes
from paper_2309_03523_b200 import _native
lib = _native.lib()
fn(); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (256 * 8))()
lib.dgc_debug_lstm_timestamps(buf, 256 * 8)
ts = np.array(buf[:L * 3], dtype=np.float64).reshape(L, 3)
t0 = ts[0, 0]
for t in range(1, 6):
    print(f"t={t} start {(ts[t,0]-t0)/1e3:8.2f} acc_ready {(ts[t,1]-t0)/1e3:8.2f} epi_done {(ts[t,2]-t0)/1e3:8.2f} us")
print("mean per-step: wait-acc", np.mean(ts[1:,1]-ts[1:,0])/1e3, "epi", np.mean(ts[1:,2]-ts[1:,1])/1e3, "step", np.mean(np.diff(ts[:,0]))/1e3)
