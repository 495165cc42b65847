# K1 with the L2::256B row-load hint (in-tree lib) vs the previous build (lib/ab)
mkdir -p gpurun_out
for lib in paper_2309_03523_b200/lib/ab/libdgc_b200.so paper_2309_03523_b200/lib/libdgc_b200.so; do
  for cfg in c2 c3; do DGC_LIB_PATH=$lib timeout 300 python tools/time_spmm_modes.py $cfg 128 2>&1 | tail -2 | sed "s|^|$(basename $(dirname $lib)) |"; done
done | tee gpurun_out/r2k_spmm_ab.txt
for lib in paper_2309_03523_b200/lib/ab/libdgc_b200.so paper_2309_03523_b200/lib/libdgc_b200.so paper_2309_03523_b200/lib/ab/libdgc_b200.so paper_2309_03523_b200/lib/libdgc_b200.so; do
  DGC_LIB_PATH=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('$(basename $(dirname $lib))', 'c2 epoch', round(d['ms_per_step'],4), 'spmm', {n: round(v['ms_per_step']*1e3,1) for n,v in k.items() if 'spmm' in n})"
done | tee -a gpurun_out/r2k_spmm_ab.txt
