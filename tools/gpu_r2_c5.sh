# C5 (10M x 128, natively generated graph, single-device restatement of the D=8 plan) + C3 lines,
# and ncu of the C5 SpMM
mkdir -p gpurun_out
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --detail > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --cpu-sample-s 40 --detail > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.err
for f in c5 c3; do python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_$f.json').read().strip().splitlines()[-1])
print('$f', d['config']['workload'][:80], round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,2), 'M edges/s; e2e', round(d['e2e']['ms_per_step'],3), 'ms; roofline', d['roofline']['kernel'], round(d['roofline']['frac'],3))
ks=sorted(d['kernels'].items(), key=lambda kv:-kv[1]['ms_per_step'])[:8]
[print('   ', k, round(v['ms_per_step']*1e3,1), 'us', round(v['GBps'])) for k,v in ks]
" || tail -5 gpurun_out/r2_bench_$f.err; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_csr -s 3 -c 1 -o gpurun_out/r2_spmm_c5 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/ncu_spmm_c5.log 2>&1
ncu -i gpurun_out/r2_spmm_c5.ncu-rep --page raw --csv > gpurun_out/r2_spmm_c5_raw.csv 2>/dev/null
ls -la gpurun_out/r2_spmm_c5*
