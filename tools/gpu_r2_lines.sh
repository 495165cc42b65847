# round-2 bench lines on one B200: C1, C3 (with the CPU oracle baseline), the
# C2 D=8 plan as 8 virtual devices (exchange data plane), C4 stale sweep
mkdir -p gpurun_out
python bench.py --config c1 --F 16 --H 16 --steps 10 --warmup 3 > gpurun_out/r2_bench_c1.json 2> gpurun_out/r2_bench_c1.err
python bench.py --config c3 --steps 5 --warmup 3 --cpu-sample-s 40 --detail > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.err
python bench.py --config c2d8 --steps 5 --warmup 3 --no-cpu-baseline --no-graph --detail > gpurun_out/r2_bench_c2d8.json 2> gpurun_out/r2_bench_c2d8.err
for f in c1 c3 c2d8; do python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_$f.json').read().strip().splitlines()[-1])
print('$f', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,2), 'M edges/s; e2e', round(d['e2e']['ms_per_step'],3), 'ms; cpu', d.get('cpu_baseline'), 'exchange', d.get('exchange'))
" || tail -5 gpurun_out/r2_bench_$f.err; done
