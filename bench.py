"""Benchmark of the B200 chunk-partitioned DGNN training step (one JSON line).

metric (BASELINE.json): DGNN train epoch time & edges/s (plus the SpMM GB/s in
the per-kernel table). One "step" = one full-batch training epoch over all T
snapshots: fwd (2 GCN layers, 2 LSTM layers) + loss + bwd + exchange +
all-reduce + optimizer. Workload at N=1: BASELINE config[1] =
synthetic 200k instances x 32 snapshots, power-law, GCN+LSTM (MPNN-LSTM),
chunk fusion, 1 B200 (artifacts/c2, the reference planner's own plan).
N>1 (torchrun, NCCL): the same graph re-planned by the reference for N
devices (artifacts/c2d{N}); strong scaling.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DGNN train epoch time & edges/sec at 1/2/4/8 B200 vs host-CPU ref; SpMM GB/s"
UNIT = "edges/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp32"])
    ap.add_argument("--F", type=int, default=128)
    ap.add_argument("--H", type=int, default=128)
    ap.add_argument("--C", type=int, default=16)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--detail", action="store_true", help="per-shape kernel table on stderr")
    ap.add_argument("--cpu-sample-s", type=float, default=25.0)
    ap.add_argument("--no-graph", action="store_true", help="eager epochs (no CUDA graph replay)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
        except (ValueError, KeyError, TypeError):
            pass
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons during the timed region, polled through
    NVML every 5 ms (nvidia-smi's query fields: clocks.sm, clocks.max.sm,
    clocks_event_reasons.*)."""

    HW_SLOWDOWN = 0x8
    SW_THERMAL = 0x20
    HW_THERMAL = 0x40
    SW_POWER_CAP = 0x4

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.max_mhz = None
            return self

        def run():
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, rs))
                except Exception:
                    pass
                self._stop.wait(0.005)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        names = {self.HW_SLOWDOWN: "hw_slowdown", self.HW_THERMAL: "hw_thermal_slowdown",
                 self.SW_THERMAL: "sw_thermal_slowdown", self.SW_POWER_CAP: "sw_power_cap"}
        reasons = sorted({n for _, rs in self.samples for bit, n in names.items() if rs & bit})
        sm = [s for s, _ in self.samples]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "sm_min_mhz": min(sm)}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload(args, pa, cfg) -> str:
    """config.workload: byte-identical in both arms (same plan, same model)."""
    sigma = "2mu" if args.config.startswith("c5") else "mu"
    model = (f"EvolveGCN-O (2 GCN, per-snapshot weights), F={cfg.F} H={cfg.H} "
             if cfg.model == "evolve" else
             f"{cfg.n_rnn}-layer {cfg.rnn.upper()} + 2 GCN, F={cfg.F} H={cfg.H} ")
    return (f"{args.config}: {pa.n_instances} instances x {pa.T} snapshots, "
            f"{pa.n_spatial_edges} edges (power-law, sigma={sigma}), {model}C={cfg.C}, "
            f"chunk plan of the reference planner ({'fused' if pa.fused else 'unfused'}, "
            f"D={pa.n_devices})")


def load_plan(args, world):
    from paper_2309_03523_b200 import load_plan_npz, single_device
    if world == 1:
        p = ROOT / "artifacts" / args.config / "plan.npz"
        if not p.exists() and (ROOT / "artifacts" / f"{args.config}d8" / "plan.npz").exists():
            # same graph, every chunk on device 0 (numerics are fusion-invariant)
            pa = single_device(load_plan_npz(ROOT / "artifacts" / f"{args.config}d8" / "plan.npz"))
            pa.meta["note"] = "single-device restatement of the D=8 plan"
            return pa, "strong"
        return load_plan_npz(p), "strong"
    # N ranks: the reference planner's D = N plan of the same graph, one shard
    # per rank (strong scaling: the graph is fixed, sim.py:76-105 n_devices = N)
    for p in (ROOT / "artifacts" / f"{args.config}d{world}" / "plan.npz",
              ROOT / "artifacts" / args.config / "plan.npz"):
        if p.exists():
            pa = load_plan_npz(p)
            if pa.n_devices == world:
                return pa, "strong"
    raise SystemExit(f"bench.py: no {world}-device plan of {args.config} "
                     f"(artifacts/{args.config}d{world}/plan.npz; tools/make_artifacts.py)")


def model_cfg(args, pa):
    from paper_2309_03523_b200 import DGNNConfig
    return DGNNConfig.for_profile(pa.profile, F=args.F, H=args.H, C=args.C,
                                  precision=args.precision, optimizer="adam", lr=1e-3)


# -- CPU baseline: the fp64 oracle port on the host cores ---------------------

def cpu_oracle(pa, cfg):
    """The CPU oracle trainer (oracle/dgnn.py, numpy fp64, all host BLAS
    threads) on the same plan and model, with its per-device layouts from the
    independent Python restatement oracle/layout.py (no product code: the
    native library is never loaded on this arm)."""
    import oracle.dgnn as od
    from oracle.layout import build_layouts
    from paper_2309_03523_b200.model import init_params, synthetic_inputs
    X, y = synthetic_inputs(pa.n_instances, cfg.F, cfg.C, 0)
    lays = build_layouts(pa.n_instances, pa.inst_entity, pa.inst_t, pa.spatial_edges,
                         pa.temporal_links, pa.structure_device, pa.chunk_of, pa.n_devices,
                         pa.group_device, pa.group_ptr, pa.group_chunks)
    T = int(pa.inst_t.max())
    ocfg = od.OracleConfig(F=cfg.F, H=cfg.H, C=cfg.C, rnn=cfg.rnn, n_rnn=cfg.n_rnn,
                           model=cfg.model, T=T, optimizer="adam", lr=1e-3)
    return od.OracleDGNN(lays, X, y, init_params(cfg, 0), ocfg, inst_t=pa.inst_t)


def cpu_epoch_time(pa, cfg, budget_s):
    """Full CPU-oracle epochs, bounded by budget_s (at most 3): min seconds."""
    orc = cpu_oracle(pa, cfg)
    times = []
    t_start = time.perf_counter()
    r = 0
    while True:
        r += 1
        t0 = time.perf_counter()
        orc.epoch(r)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start + times[-1] > budget_s or r >= 3:
            break
    return min(times), r


def run_reference(args):
    """Reference arm: the CPU oracle port of the path on the host cores (rank 0
    only; other ranks exit). One step = one full fp64 epoch of the same plan
    (the D = N plan at N ranks) and model as our arm."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    pa, scaling = load_plan(args, world)
    cfg = model_cfg(args, pa)
    cores = os.cpu_count()
    t_build = time.perf_counter()
    orc = cpu_oracle(pa, cfg)
    t_build = time.perf_counter() - t_build
    times = []
    for r in range(1, args.warmup + args.steps + 1):
        t0 = time.perf_counter()
        orc.epoch(r)
        times.append(time.perf_counter() - t0)
    times = times[args.warmup:] or times
    ep = statistics.mean(times)
    value = pa.n_spatial_edges / ep
    loaded = [Path(l.split()[-1]).name for l in Path("/proc/self/maps").read_text().splitlines()
              if "libdgc_b200" in l] if Path("/proc/self/maps").exists() else []
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ep * 1e3, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args, pa, cfg), "parallelism": "host CPU"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "cpu_model": cpu_model(), "epoch_s": ep,
                             "sample": f"{args.steps} full epochs (after {args.warmup} warm-up) "
                                       "of the fp64 oracle (oracle/dgnn.py) on the same plan/"
                                       "model, layouts from oracle/layout.py "
                                       f"({t_build:.0f} s to build, untimed); the reference "
                                       "(dynpart) has no DGNN trainer",
                             "native_libs_loaded": sorted(set(loaded))},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# -- our arm -------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2309_03523_b200 import ops
    from paper_2309_03523_b200.model import synthetic_inputs
    from paper_2309_03523_b200.trainer import DGNNTrainer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DGC_BENCH_BACKEND=gloo + DGC_BENCH_ONE_GPU=1: smoke-test the N>1 code
    # path with every rank on cuda:0 (a one-GPU box); the real run is NCCL
    gpu = 0 if os.environ.get("DGC_BENCH_ONE_GPU") == "1" else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        backend = os.environ.get("DGC_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    pa, scaling = load_plan(args, world)
    cfg = model_cfg(args, pa)
    X, y = synthetic_inputs(pa.n_instances, cfg.F, cfg.C, 0)
    distributed = world > 1 and scaling == "strong"
    # single-device epochs replay one captured CUDA graph (same kernels, no
    # per-launch host latency); multi-rank epochs have host-side count syncs
    tr = DGNNTrainer(pa, cfg, None, seed=0, device=dev, distributed=distributed, features=X,
                     labels=y, cuda_graph=not args.no_graph)
    sh = tr.shards[0]
    flush = torch.empty(320 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        tr.run_epoch()
    # ---- device-timed region (inputs resident in HBM) ----
    times = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            rep = tr.run_epoch()  # brackets the step with CUDA events (wall_ms)
            times.append(rep.wall_ms)
            rep_last = rep
            barrier()
    # ---- per-kernel table: separate eager epochs with CUDA events around every
    # native launch on its stream (never inside the timed region) ----
    ops._prof_detail = True  # per-shape names: the dominant kernel is one (kernel, shape)
    prof = ops.profile()
    graph_mode, tr.cuda_graph = tr.cuda_graph, False
    n_prof = max(1, min(args.steps, 3))
    if distributed:
        tr.runner.comm_timing = []
    with prof:
        for _ in range(n_prof):
            flush.zero_()
            barrier()
            tr.run_epoch()
            barrier()
    tr.cuda_graph = graph_mode
    exchange = None
    if distributed:
        # payload all-to-allvs on the comm stream (overlapped with compute), per
        # step; NVLink 5 = 900 GB/s per direction per GPU
        ct = tr.runner.comm_timing
        tr.runner.comm_timing = None
        torch.cuda.synchronize()
        x_ms = sum(a.elapsed_time(b) for a, b, _, _ in ct) / n_prof
        x_out = sum(o for _, _, o, _ in ct) / n_prof
        x_in = sum(i for _, _, _, i in ct) / n_prof
        t = torch.tensor([x_ms, x_out, x_in], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        x_ms, x_out, x_in = t.tolist()
        gbs = max(x_out, x_in) / (x_ms / 1e3) / 1e9 if x_ms > 0 else 0.0
        exchange = {"bytes_out_per_step": x_out, "bytes_in_per_step": x_in,
                    "a2a_ms_per_step": x_ms, "GBps": gbs, "peak_GBps": 900.0,
                    "frac": gbs / 900.0,
                    "note": "busiest rank; NCCL all-to-allv time on the comm stream, which "
                            "overlaps interior-row SpMM (not on the critical path when hidden)"}
    # per-step averages over the profiled epochs, expressed per `steps` epochs
    kern = {k: {f: v[f] * args.steps / n_prof for f in ("ms", "launches", "kernels", "bytes", "flops")}
            for k, v in prof.summary().items()}
    step_ms = float(np.mean(times))
    if world > 1:
        t = torch.tensor([step_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms = float(t.item())
    edges_total = pa.n_spatial_edges * (world if scaling == "weak" else 1)
    value = edges_total / (step_ms / 1e3)
    # ---- end-to-end through the public API with host buffers: every step
    # installs inputs copied from pinned host memory (the next step's copy runs
    # on a copy stream during this step: trainer.stage_inputs) and reads its
    # loss back to the host. Software-pipelined like a training loop: step i+1
    # is submitted before step i's loss is read, so the host read overlaps the
    # device; the timed region covers K submissions, K H2D copies and K loss
    # reads (the last read and every queued copy drained before the end event).
    xs, ys = tr.host_inputs(X, y)
    tr.stage_inputs(xs, ys)

    def pipelined(k):
        prev = None
        for _ in range(k):
            p = tr.submit_epoch(next_inputs=(xs, ys))
            if prev is not None:
                float(prev.result().loss)  # D2H read of the step result
            prev = p
        float(prev.result().loss)
        torch.cuda.synchronize()

    pipelined(args.warmup)
    barrier()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    pipelined(args.steps)
    e.record()
    barrier()
    e2e_ms = [s.elapsed_time(e) / args.steps]
    e2e_step = float(np.mean(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_step], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_step = float(t.item())
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    hbm, tflops, src = peaks()
    # DRAM traffic of the dominant kernel from the committed ncu --set full
    # capture of this workload (profiles/ncu_traffic.json), per launch
    traffic = None
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists():
        rec = json.loads(tp.read_text()).get("kernels", {})
    top = max(kern.items(), key=lambda kv: kv[1]["ms"])
    name, d = top
    base = name.split("[")[0]
    # the ncu capture's shape must be the dominant one for its traffic to apply
    key = f"{args.config}/{base}"  # records are per workload (config) and shape
    if tp.exists() and key in rec and rec[key].get("shape", name) == name:
        traffic = rec[key]["traffic_bytes"]
    avg_ms = d["ms"] / d["launches"]
    achieved = (d["bytes"] / d["launches"]) / (avg_ms / 1e3) / 1e9
    per_kernel = {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                      "GBps": (v["bytes"] / v["launches"]) / (v["ms"] / v["launches"] / 1e3) / 1e9,
                      "TFLOPs": (v["flops"] / v["launches"]) / (v["ms"] / v["launches"] / 1e3) / 1e12}
                  for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["ms"])}
    gpu_launches = int(sum(v["kernels"] for v in kern.values()) / args.steps)
    if args.detail:
        for k, v in per_kernel.items():
            print(f"{k:48s} {v['ms_per_step']*1e3:9.1f} us/step  x{v['launches_per_step']:.0f}  "
                  f"{v['GBps']:8.1f} GB/s {v['TFLOPs']:7.2f} TF/s", file=sys.stderr)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        t_cpu, n_ep = cpu_epoch_time(pa, cfg, args.cpu_sample_s)
        cpu = {"value": pa.n_spatial_edges / t_cpu, "unit": UNIT, "cores": os.cpu_count(),
               "kind": "port", "epoch_s": t_cpu, "cpu_model": cpu_model(),
               "sample": f"{n_ep} full epoch(s) of the fp64 numpy oracle (oracle/dgnn.py) on the "
                         f"same plan and model, all host BLAS threads"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "tf32" if args.precision == "tf32" else "f32",
        "data": "synthetic",
        "config": {"workload": workload(args, pa, cfg),
                   "epoch_ms": step_ms, "l2": "flushed (320 MB write) before every timed step",
                   "parallelism": f"chunk-sharded x{world}" if distributed else
                   ("replicas" if world > 1 else "1 GPU")},
        "e2e": {"value": edges_total / (e2e_step / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(sum(x.numel() * x.element_size() + t.numel() * t.element_size()
                                              for x, t in zip(xs, ys))),
                "pipeline": ("inputs double-buffered: step i+1's H2D overlaps step i (4 concurrent copy streams: one pinned stream moved 26-55 GB/s on these boxes, four 45+); "
                             + ("TF32 mode consumes in-range features at fp16 precision and ships "
                                "them as fp16 (bit-identical to on-device rounding); the host-side "
                                "fp32->fp16 conversion happens once, outside the timed region"
                                if sh.x_f16 else
                                "TF32 mode ships the TF32-rounded features as their 3 significant "
                                "bytes (bit-identical to on-device rounding); the host-side packing "
                                "happens once, outside the timed region")),
                "d2h_bytes_per_step": 8, "ms_per_step": e2e_step,
                "loop": ("software-pipelined: step i+1 submitted before step i's loss is read "
                         "(trainer.submit_epoch); time = K steps / K"),
                "l2": "not flushed between pipelined steps; per-step working set (> 2 GB) >> 126 MB L2"},
        "roofline": {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                     "peak_source": src, "algorithmic_bytes_per_launch": d["bytes"] / d["launches"],
                     "avg_launch_ms": avg_ms},
        "kernels": per_kernel,
        "gpu_launches": gpu_launches,
        "exchange": exchange,
        "epoch_report": {"per_device_compute_ms": rep_last.per_device_compute_ms,
                         "per_device_wall_ms": rep_last.per_device_wall_ms,
                         "load_divergence": rep_last.load_divergence,
                         "spatial_traffic_bytes": rep_last.spatial_traffic_bytes,
                         "temporal_traffic_bytes": rep_last.temporal_traffic_bytes,
                         "exchanged_bytes": rep_last.exchanged_bytes},
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def spawn(args) -> int:
    """`python bench.py --gpus N` without a launcher: re-run this script under
    torchrun, one rank per GPU (rendezvous on 127.0.0.1); rank 0 prints the
    line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(a))
    if int(os.environ.get("WORLD_SIZE", "1")) != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}")
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
