timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "lstm_bwd" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_trainer.py -q -x 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --detail > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_q.json").read().strip().splitlines()[-1])
print("epoch ms", round(d["ms_per_step"], 4), "e2e ms", round(d["e2e"]["ms_per_step"], 4))
for k, v in sorted(d["kernels"].items(), key=lambda kv: -kv[1]["ms_per_step"])[:4]:
    print(f"  {k:55s} {v['ms_per_step']*1e3:8.1f} us")
PY
DGC_BPTT_KSPLIT=1 timeout 300 python bench.py --no-cpu-baseline --detail > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_k.json").read().strip().splitlines()[-1])
print("KSPLIT epoch ms", round(d["ms_per_step"], 4))
for k, v in sorted(d["kernels"].items(), key=lambda kv: -kv[1]["ms_per_step"])[:2]:
    print(f"  {k:55s} {v['ms_per_step']*1e3:8.1f} us")
PY
