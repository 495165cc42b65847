"""Per-position timing of the fused-projection LSTM forward (C2 shape)."""
# per-position timestamps need a build with them compiled in: make clean && make DGC_TS=1
import ctypes
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2309_03523_b200 import ops, _native
from paper_2309_03523_b200.layout import pack_sequences_native
H = 128
lengths = np.full(6250, 32)
seq, pos, mask, _ = pack_sequences_native(lengths)
R, L = seq.shape
offs = np.concatenate([[0], np.cumsum(lengths)])
n = int(offs[-1])
slot_row = np.where(seq >= 0, offs[np.maximum(seq, 0)] + pos, -1).astype(np.int32).reshape(-1)
dev = "cuda"
x = torch.randn((n, H), device=dev); WxT = torch.randn((4 * H, H), device=dev) / H ** 0.5
Ut = torch.randn((4 * H, H), device=dev) / H ** 0.5; b = torch.zeros(4 * H, device=dev)
sr = torch.tensor(slot_row, device=dev); sm = torch.tensor(mask.reshape(-1), device=dev)
sc = torch.full((R * L,), -1, dtype=torch.int32, device=dev); carry = torch.zeros((1, 2 * H), device=dev)
hc = torch.zeros((n, 2 * H), device=dev); save = torch.zeros((n, 7 * H), device=dev)
x16 = x.half(); Wx = WxT.t().contiguous(); U = Ut.t().contiguous()
fn = lambda: ops.lstm_fwd_tc_f16x(x16, Wx, U, b, sr, sm, sc, carry, R, L, H, 2 * H, hc, hc[:, H:], save)
fn(); torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3): fn()
e.record(); torch.cuda.synchronize()
print(f"fused fwd H {H}: {s.elapsed_time(e) / 3:.3f} ms")
fn(); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (256 * 16))()
_native.lib().dgc_debug_lstm_timestamps(buf, 256 * 16)
ts = np.array(buf[:L * 8], dtype=np.float64).reshape(L, 8)
print("per-step us: h-ready->acc", np.mean(ts[:, 1] - ts[:, 0]) / 1e3, "epi", np.mean(ts[:, 2] - ts[:, 1]) / 1e3,
      "epi_end->next h-ready", np.mean(ts[1:, 0] - ts[:-1, 2]) / 1e3, "step", np.mean(np.diff(ts[:, 0])) / 1e3)
ch = [ts[:, 1], ts[:, 3], ts[:, 4], ts[:, 5], ts[:, 2]]
print("per-chunk epilogue us:", [round(float(np.mean(ch[i + 1] - ch[i])) / 1e3, 2) for i in range(4)])
print("MMA warp (us rel. to h-ready[p]): x-part issued for p (before h-ready)", np.mean(ts[:, 6] - ts[:, 0]) / 1e3,
      "U kb2 ready", np.mean(ts[:, 7] - ts[:, 0]) / 1e3, "acc ready", np.mean(ts[:, 1] - ts[:, 0]) / 1e3)
for p in range(1, 6):
    print(p, " ".join(f"{(ts[p, k] - ts[p, 0]) / 1e3:6.2f}" for k in (6, 0, 7, 1, 3, 4, 5, 2)))
t2 = np.array(buf[256 * 8:256 * 8 + L * 8], dtype=np.float64).reshape(L, 8)
d = np.diff(t2[1:, :6], axis=1) / 1e3
print("chunk 0 (us): tmem ld", d[:, 0].mean(), "stage+lds", d[:, 1].mean(), "math", d[:, 2].mean(),
      "stores", d[:, 3].mean(), "put_h", d[:, 4].mean())
wb = (ctypes.c_ulonglong * (256 * 32))()
_native.lib().dgc_debug_lstm_timestamps_warps(wb, 256 * 32)
w = np.array(wb, dtype=np.float64).reshape(256, 32)
k0 = w[2, 30]
print(f"kernel (CTA0, us after setup): prologue done {(w[2,31]-k0)/1e3:.2f}, first h-ready {(ts[0,0]-k0)/1e3:.2f}, "
      f"first acc {(ts[0,1]-k0)/1e3:.2f}, last epilogue done {(ts[L-1,2]-k0)/1e3:.2f}, "
      f"before exit sync {(w[3,30]-k0)/1e3:.2f}, after {(w[3,31]-k0)/1e3:.2f}")
