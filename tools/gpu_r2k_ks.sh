# split-K of the concurrent stacked weight-gradient GEMM (C2 epoch), 2 runs each
mkdir -p gpurun_out
for v in 0 74 37 0 74 37 111; do
  DGC_STACKED_KSPLIT=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('ks=$v c2 epoch', round(d['ms_per_step'],4), {n: round(v['ms_per_step']*1e3,1) for n,v in k.items() if 'stacked' in n or '512 a0b0' in n})"
done | tee gpurun_out/r2k_ks.txt
DGC_STACKED_KSPLIT=74 timeout 900 python -m pytest tests/test_gpu_c2_parity.py -m gpu -x -q 2>&1 | tail -2
