# per-kernel C2 epoch times under GEMM tuning environment variables
run() {
  env "$@" timeout 300 python bench.py --no-cpu-baseline --detail --steps 40 > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err
  python - "$@" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/bench_e.json").read().strip().splitlines()[-1])
g = {k: v["ms_per_step"] * 1e3 for k, v in d["kernels"].items() if k.startswith("gemm")}
print(" ".join(sys.argv[1:]) or "default", "epoch", round(d["ms_per_step"], 4), "gemm total", round(sum(g.values()), 1))
for k, v in sorted(g.items(), key=lambda kv: -kv[1])[:5]:
    print(f"   {k:50s} {v:7.1f}")
PY
}
run X=1
run DGC_GEMM_MAX_STAGES=6
run DGC_GEMM_MAX_STAGES=8
run DGC_GEMM_MAX_STAGES=8 DGC_GEMM_ONE_BOX=1
