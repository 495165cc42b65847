# concurrent LSTM weight-/input-gradient GEMM CTA splits (C2 epoch), 2 runs each
for c in 0 74,74 0 74,74 84,64 64,84; do
  DGC_CONC_BWD=$c timeout 300 python bench.py --no-cpu-baseline --steps 40 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
  python -c "
import json
d = json.loads(open('gpurun_out/bench_c.json').read().strip().splitlines()[-1])
print('$c', 'epoch', round(d['ms_per_step'], 4), 'e2e', round(d['e2e']['ms_per_step'], 4))
" || tail -3 gpurun_out/bench_c.err
done
