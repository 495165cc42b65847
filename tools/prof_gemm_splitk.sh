out=gpurun_out/prof_gemm; mkdir -p $out
for idx in 7 13; do
  timeout 600 ncu --set full --clock-control none -k regex:gemm_tf32 -s $idx -c 1 -o $out/g$idx \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph > $out/log$idx 2>&1
  ncu -i $out/g$idx.ncu-rep --page raw --csv > $out/g${idx}_raw.csv 2>/dev/null
done
ls $out
