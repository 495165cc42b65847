# fp16 dh_out A/B + parity, and the random-row gather ceiling probe
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "lstm_bwd" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_c2_parity.py tests/test_gpu_trainer.py -m gpu -x -q 2>&1 | tail -3
for v in 0 1 0 1; do
  DGC_DH16=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('dh16=$v c2 epoch', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), {n: round(v['ms_per_step']*1e3,1) for n,v in k.items() if 'lstm' in n or '512 a0b0' in n or 'x16 a0b1' in n})"
done | tee gpurun_out/r2i_dh16_ab.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/row_gather tools/probes/row_gather.cu && timeout 300 /tmp/row_gather | tee gpurun_out/r2i_row_gather.txt
