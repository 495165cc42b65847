# C5 (10M x 128, natively generated graph, single-device restatement of the D=8 plan)
mkdir -p gpurun_out
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --detail > gpurun_out/r2h_bench_c5.json 2> gpurun_out/r2h_bench_c5.err
python -c "
import json; d=json.loads(open('gpurun_out/r2h_bench_c5.json').read().strip().splitlines()[-1])
print('c5', d['config']['workload'][:80], round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,2), 'M edges/s; e2e', round(d['e2e']['ms_per_step'],3), 'ms; roofline', d['roofline']['kernel'], round(d['roofline']['frac'],3))
ks=sorted(d['kernels'].items(), key=lambda kv:-kv[1]['ms_per_step'])[:8]
[print('   ', k, round(v['ms_per_step']*1e3,1), 'us', round(v['GBps'])) for k,v in ks]
" || tail -5 gpurun_out/r2h_bench_c5.err
