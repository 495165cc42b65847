# bench lines for the other BASELINE configs (not the headline): C1 and C3 on one B200
python bench.py --config c1 --F 16 --H 16 --steps 10 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
for f in c1 c3; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json'))
print('$f', d['config']['workload'], round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,2), 'M edges/s e2e', round(d['e2e']['ms_per_step'],3), 'cpu', d.get('cpu_baseline'))
" || tail -5 gpurun_out/bench_$f.err; done
