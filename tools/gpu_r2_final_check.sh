# final state check: GPU suite, smoke, default bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_final_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/r2_final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r2_final_bench_c2.json 2> gpurun_out/r2_final_bench_c2.err
python -c "
import json; d=json.loads(open('gpurun_out/r2_final_bench_c2.json').read().strip().splitlines()[-1])
print('c2', round(d['ms_per_step'],4), 'ms', round(d['value']/1e6,1), 'M edges/s; e2e', round(d['e2e']['ms_per_step'],4), 'launches', d['gpu_launches'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'])"
