# K1 variant sweep (DGC_SPMM_MODE) at C2 and C3, then the re-entry check
mkdir -p gpurun_out
for cfg in c2 c3; do for m in 0 2 4 24 44; do
  DGC_SPMM_MODE=$m timeout 300 python tools/time_spmm_modes.py $cfg 128 2>&1 | tail -2
done; done | tee gpurun_out/r2i_spmm_modes.txt
for m in 0 2 24; do
  DGC_SPMM_MODE=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('mode $m c2 epoch', round(d['ms_per_step'],4), 'spmm', {n: round(v['ms_per_step']*1e3,1) for n,v in k.items() if 'spmm' in n})"
done | tee -a gpurun_out/r2i_spmm_modes.txt
bash tools/gpu_r2i_check.sh
