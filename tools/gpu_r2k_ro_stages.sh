# fused readout with 4 h16 stages (in-tree lib) vs 3 (lib/ab): C2 and C3 epochs, readout parity
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "fused_readout" 2>&1 | tail -1
for cfg in c2 c3; do for lib in paper_2309_03523_b200/lib/ab/libdgc_b200.so paper_2309_03523_b200/lib/libdgc_b200.so paper_2309_03523_b200/lib/ab/libdgc_b200.so paper_2309_03523_b200/lib/libdgc_b200.so; do
  DGC_LIB_PATH=$lib timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('$cfg', '$(basename $(dirname $lib))', 'epoch', round(d['ms_per_step'],4), {n: round(v['ms_per_step']*1e3,1) for n,v in k.items() if 'readout' in n})"
done; done | tee gpurun_out/r2k_ro_stages.txt
