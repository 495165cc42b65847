# fused fp16 readout: kernel parity, trainer parity, A/B bench
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "fused_readout" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_c2_parity.py tests/test_gpu_trainer.py -m gpu -x -q 2>&1 | tail -5
for v in 0 1 0 1; do
  DGC_FUSED_READOUT=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('fused=$v c2 epoch', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), {n: round(v['ms_per_step']*1e3,1) for n,v in k.items() if 'readout' in n or 'softmax' in n or 'x16 ' in n or '16x128' in n or '128x16' in n or 'reduce' in n})"
done | tee gpurun_out/r2i_readout_ab.txt
