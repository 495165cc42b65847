"""bench.py's JSON contract (both arms) on the small C1 configuration: every
key the driver reads is present and sane."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _line(*args):
    out = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--F", "16", "--H", "16",
                          "--steps", "2", "--warmup", "3", *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_ours_contract():
    d = _line("--cpu-sample-s", "2")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "roofline", "cpu_baseline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["n_gpus"] == 1 and d["steps"] == 2
    assert d["higher_is_better"] is True and d["unit"] == "edges/s"
    assert "workload" in d["config"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert 0 < d["roofline"]["frac"] < 1.5
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    assert d["gpu_launches"] > 10
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_bench_reference_contract():
    d = _line("--impl", "reference")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "edges/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
    # independent of the product: the native library is never mapped on this arm,
    # and both arms name the same workload byte for byte
    assert d["cpu_baseline"]["native_libs_loaded"] == []
    assert d["config"]["workload"] == _line("--cpu-sample-s", "1")["config"]["workload"]


def test_bench_gpus_n_spawns_ranks():
    """`bench.py --gpus 2` without a launcher re-runs itself under torchrun with
    one rank per GPU (here both ranks on cuda:0 over gloo: a one-GPU box) on
    the reference planner's 2-device plan; rank 0 prints one line."""
    import os
    env = dict(os.environ, DGC_BENCH_ONE_GPU="1", DGC_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    for impl in ("ours", "reference"):
        out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "t2",
                              "--F", "16", "--H", "16", "--steps", "2", "--warmup", "3",
                              "--impl", impl], cwd=ROOT, capture_output=True, text=True,
                             timeout=900, env=env)
        assert out.returncode == 0, out.stderr[-3000:]
        lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1, out.stdout
        d = json.loads(lines[0])
        assert d["n_gpus"] == 2 and d["value"] > 0
        if impl == "ours":
            assert d["config"]["parallelism"] == "chunk-sharded x2"
            assert d["scaling"] == "strong"
        else:
            assert d["impl"] == "reference"
            assert d["cpu_baseline"]["native_libs_loaded"] == []
