"""C4: adaptive stale aggregation sweep (BASELINE.json config 4).

Trains the chunk-partitioned DGNN on a D-device reference plan (default: the
200k-instance C2 graph planned for 8 devices, artifacts/c2d8) with every
staleness setting -- off, "staleness bound" b = 0..8 mapped to
StaleConfig.static(b/10), adaptive-relax and
adaptive-tighten -- and reports boundary-exchange bytes (reference-billed and
actually moved) against the loss / accuracy delta versus staleness off.

Labels come from a fixed random linear teacher on the input features so that
accuracy is meaningful. Runs the D shards as virtual devices on one GPU
(LocalRunner: same kernels and exchange logic as the NCCL path).

  python tools/stale_sweep.py [--plan c2d8] [--epochs 30] [--H 64]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2309_03523_b200 import DGNNConfig, StaleConfig, load_plan_npz  # noqa: E402
from paper_2309_03523_b200.model import init_params, synthetic_inputs  # noqa: E402
from paper_2309_03523_b200.trainer import DGNNTrainer  # noqa: E402


def teacher_labels(X, C, seed=11):
    W = np.random.default_rng(seed).standard_normal((X.shape[1], C)).astype(np.float32)
    return np.argmax(X @ W, axis=1).astype(np.int32)


def accuracy(tr):
    hit = tot = 0
    for sh in tr.shards:
        pred = sh.logits.argmax(dim=1).to(torch.int32)
        hit += int((pred == sh.y).sum().item())
        tot += sh.y.numel()
    return hit / tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan", default="c2d8")
    ap.add_argument("--epochs", type=int, default=30)
    ap.add_argument("--H", type=int, default=64)
    ap.add_argument("--F", type=int, default=32)
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r1_stale_sweep.json"))
    args = ap.parse_args()
    pa = load_plan_npz(ROOT / "artifacts" / args.plan / "plan.npz")
    cfg = DGNNConfig.for_profile(pa.profile, F=args.F, H=args.H, C=8, precision="tf32",
                                 optimizer="adam", lr=args.lr)
    X, _ = synthetic_inputs(pa.n_instances, cfg.F, cfg.C, 0)
    y = teacher_labels(X, cfg.C)
    params = init_params(cfg, 0)
    settings = [("off", StaleConfig.off())]
    settings += [(f"bound{b}", StaleConfig.static(b / 10)) for b in range(9)]
    settings += [("adaptive-relax", StaleConfig.adaptive()),
                 ("adaptive-tighten", StaleConfig.adaptive(True))]
    results = []
    for name, scfg in settings:
        tr = DGNNTrainer(pa, cfg, scfg, seed=0, features=X, labels=y, params=params)
        t0 = time.time()
        billed = moved = full = 0
        hist = []
        for _ in range(args.epochs):
            rep = tr.run_epoch()
            billed += rep.spatial_traffic_bytes + rep.temporal_traffic_bytes
            moved += rep.exchanged_bytes
            full += rep.stale_sent_bytes + rep.stale_avoided_bytes if name != "off" else (
                rep.spatial_traffic_bytes + rep.temporal_traffic_bytes)
            hist.append(rep.loss)
        acc = accuracy(tr)
        results.append(dict(setting=name, final_loss=hist[-1], train_acc=acc,
                            billed_bytes=billed, moved_bytes=moved, loss_curve=hist,
                            wall_s=time.time() - t0))
        print(f"{name:18s} loss {hist[-1]:.4f} acc {acc:.4f} billed {billed/1e6:9.2f} MB "
              f"moved {moved/1e6:9.2f} MB", flush=True)
    base = results[0]
    for r in results:
        r["loss_delta"] = r["final_loss"] - base["final_loss"]
        r["acc_delta"] = r["train_acc"] - base["train_acc"]
        r["billed_reduction_pct"] = 100.0 * (1 - r["billed_bytes"] / base["billed_bytes"])
        r["moved_reduction_pct"] = 100.0 * (1 - r["moved_bytes"] / base["moved_bytes"])
    meta = dict(plan=args.plan, n_instances=pa.n_instances, n_devices=pa.n_devices,
                epochs=args.epochs, model=f"2 GCN + {cfg.n_rnn}x{cfg.rnn.upper()}",
                F=cfg.F, H=cfg.H, C=cfg.C, precision=cfg.precision, gpu=torch.cuda.get_device_name())
    Path(args.out).write_text(json.dumps(dict(meta=meta, results=results), indent=1))
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
