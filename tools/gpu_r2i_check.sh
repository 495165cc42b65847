# session re-entry check on one B200: full GPU suite, smoke, default bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/r2i_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r2i_bench_c2.json 2> gpurun_out/r2i_bench_c2.err
python -c "
import json; d=json.loads(open('gpurun_out/r2i_bench_c2.json').read().strip().splitlines()[-1])
print('c2', round(d['ms_per_step'],4), 'ms e2e', round(d['e2e']['ms_per_step'],4), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'])
ks=sorted(d['kernels'].items(), key=lambda kv:-kv[1]['ms_per_step'])[:10]
[print('   ', k, round(v['ms_per_step']*1e3,1), 'us', round(v['GBps'])) for k,v in ks]
" || tail -5 gpurun_out/r2i_bench_c2.err
