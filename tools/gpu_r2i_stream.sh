# K1 streaming (cp.async ring) variants vs the row-per-sub-warp kernel at C2 / C3
mkdir -p gpurun_out
for cfg in c2 c3; do for m in 0 86 84 122 163; do
  DGC_SPMM_STREAM=$m timeout 300 python tools/time_spmm_modes.py $cfg 128 2>&1 | tail -2
done; done | tee gpurun_out/r2i_spmm_stream.txt
for m in 0 86 122; do
  DGC_SPMM_STREAM=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('stream $m c2 epoch', round(d['ms_per_step'],4), 'spmm', {n: round(v['ms_per_step']*1e3,1) for n,v in k.items() if 'spmm' in n})"
done | tee -a gpurun_out/r2i_spmm_stream.txt
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "spmm" 2>&1 | tail -3
