# K1 neighbour-row load flavours (DGC_SPMM_LD) at C2 / C3 and the C2 epoch
mkdir -p gpurun_out
for cfg in c2 c3; do for m in 0 1 2 3; do
  DGC_SPMM_LD=$m DGC_SPMM_MODE=$m timeout 300 python tools/time_spmm_modes.py $cfg 128 2>&1 | tail -2
done; done | tee gpurun_out/r2k_spmm_ld.txt
for m in 0 1 2 3; do
  DGC_SPMM_LD=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('ld $m c2 epoch', round(d['ms_per_step'],4), 'spmm', {n: round(v['ms_per_step']*1e3,1) for n,v in k.items() if 'spmm' in n})"
done | tee -a gpurun_out/r2k_spmm_ld.txt
