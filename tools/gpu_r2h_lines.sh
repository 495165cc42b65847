# round-2 final bench lines on one B200: C2 (default bench, with the CPU
# baseline), the reference arm, C1, C3
mkdir -p gpurun_out
python bench.py > gpurun_out/r2h_bench_c2.json 2> gpurun_out/r2h_bench_c2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2h_bench_reference.json 2> gpurun_out/r2h_bench_reference.err
python bench.py --config c1 --F 16 --H 16 --steps 10 --warmup 3 > gpurun_out/r2h_bench_c1.json 2> gpurun_out/r2h_bench_c1.err
python bench.py --config c3 --steps 5 --warmup 3 --cpu-sample-s 40 --detail > gpurun_out/r2h_bench_c3.json 2> gpurun_out/r2h_bench_c3.err
for f in c2 reference c1 c3; do python -c "
import json; d=json.loads(open('gpurun_out/r2h_bench_$f.json').read().strip().splitlines()[-1])
print('$f', round(d['ms_per_step'],4), 'ms', round(d['value']/1e6,2), 'M edges/s; e2e', round(d['e2e']['ms_per_step'],4) if 'ms_per_step' in d['e2e'] else d['e2e'], '; roofline', d.get('roofline'), '; cpu', d.get('cpu_baseline'), '; clocks', d.get('clocks'))
" || tail -5 gpurun_out/r2h_bench_$f.err; done
