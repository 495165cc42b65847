# round-2 final evidence (r2k) on one B200: GPU suite + smoke, bench lines
# (C2 headline with the CPU baseline, reference arm, C1, C3, C5), launch list
# and ncu --set full of the top kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2k_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/r2k_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/r2k_bench_c2.json 2> gpurun_out/r2k_bench_c2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2k_bench_reference.json 2> gpurun_out/r2k_bench_reference.err
python bench.py --config c1 --F 16 --H 16 --steps 10 --warmup 3 > gpurun_out/r2k_bench_c1.json 2> gpurun_out/r2k_bench_c1.err
python bench.py --config c3 --steps 5 --warmup 3 --cpu-sample-s 40 --detail > gpurun_out/r2k_bench_c3.json 2> gpurun_out/r2k_bench_c3.err
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --detail > gpurun_out/r2k_bench_c5.json 2> gpurun_out/r2k_bench_c5.err
for f in c2 reference c1 c3 c5; do python -c "
import json; d=json.loads(open('gpurun_out/r2k_bench_$f.json').read().strip().splitlines()[-1])
e=d.get('e2e',{})
print('$f', round(d['ms_per_step'],4), 'ms', round(d['value']/1e6,2), 'M edges/s; e2e', round(e['ms_per_step'],4) if 'ms_per_step' in e else e, '; roofline', {k: d['roofline'][k] for k in ('kernel','frac')} if d.get('roofline') else None, '; cpu', (d.get('cpu_baseline') or {}).get('value'), '; clocks', d.get('clocks'))
" || tail -5 gpurun_out/r2k_bench_$f.err; done
bash tools/gpu_profile.sh r2k readout_f16 > gpurun_out/prof_r2k.log 2>&1
head -30 gpurun_out/prof_r2k/launches_summary.txt
ls gpurun_out/prof_r2k
