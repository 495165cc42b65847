# forward LSTM gate activations two cells per MUFU op (tanh.approx.f16x2): A/B vs lib/ab, parity
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "lstm" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_c2_parity.py tests/test_gpu_trainer.py -m gpu -x -q 2>&1 | tail -3
for lib in paper_2309_03523_b200/lib/ab/libdgc_b200.so paper_2309_03523_b200/lib/libdgc_b200.so paper_2309_03523_b200/lib/ab/libdgc_b200.so paper_2309_03523_b200/lib/libdgc_b200.so; do
  DGC_LIB_PATH=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('$(basename $(dirname $lib))', 'c2 epoch', round(d['ms_per_step'],4), {n: round(v['ms_per_step']*1e3,1) for n,v in k.items() if 'lstm' in n})"
done | tee gpurun_out/r2k_gates_ab.txt
