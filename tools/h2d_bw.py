"""Pinned host->device copy bandwidth on this box (the e2e input pipeline's bound):
one stream, 2 / 4 concurrent streams, and 2 MB chunks; plus the host's NUMA view."""
import os
import subprocess
import torch

mb = 52
n = mb * (1 << 20)
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return n * reps / e0.elapsed_time(e1) / 1e6


print(f"H2D {mb} MB one stream: {timed(lambda: d.copy_(h, non_blocking=True)):.1f} GB/s")
for ns in (2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    cur = torch.cuda.current_stream()

    def multi():
        part = n // ns
        for i, s in enumerate(streams):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
    print(f"H2D {mb} MB over {ns} streams: {timed(multi):.1f} GB/s")
d2h = torch.empty(n, dtype=torch.uint8).pin_memory()
print(f"D2H {mb} MB one stream: {timed(lambda: d2h.copy_(d, non_blocking=True)):.1f} GB/s")
print("cpus:", os.cpu_count(), "gpu numa:", open("/sys/bus/pci/devices/" + subprocess.run(
    ["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True,
    text=True).stdout.strip().lower()[4:] + "/numa_node").read().strip() if True else "")
