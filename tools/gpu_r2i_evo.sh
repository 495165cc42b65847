# fused EvolveGCN readout: kernel parity, trainer parity (EvolveGCN tests), C3 A/B
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "fused_readout" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_trainer.py tests/test_gpu_c2_parity.py -m gpu -x -q 2>&1 | tail -5
for v in 0 1; do
  DGC_FUSED_READOUT=$v timeout 400 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('fused=$v c3 epoch', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), {n: round(v['ms_per_step']*1e3,1) for n,v in k.items() if 'readout' in n or 'softmax' in n or 'x16 ' in n or '16x' in n or 'x16x' in n or 'reduce' in n})"
done | tee gpurun_out/r2i_readout_evo_ab.txt
