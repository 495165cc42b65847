# round-2 ncu evidence at C2 (launch list + --set full of the top kernels) and C3/C5 SpMM
mkdir -p gpurun_out
bash tools/gpu_profile.sh r2c lstm_bwd_tc2k lstm_fwd_tc2v spmm_csr gemm_tf32_kernel > gpurun_out/prof_r2c.log 2>&1
head -22 gpurun_out/prof_r2c/launches_summary.txt
for k in lstm_bwd_tc2k lstm_fwd_tc2v spmm_csr gemm_tf32_kernel; do
  ncu -i gpurun_out/prof_r2c/$k.ncu-rep --page source --csv --print-source=sass > gpurun_out/prof_r2c/${k}_sass.csv 2>/dev/null
done
timeout 900 ncu --set full --clock-control none -k regex:spmm_csr -s 3 -c 1 -o gpurun_out/prof_r2c/spmm_c3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/prof_r2c/ncu_spmm_c3.log 2>&1
ncu -i gpurun_out/prof_r2c/spmm_c3.ncu-rep --page raw --csv > gpurun_out/prof_r2c/spmm_c3_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:spmm_csr -s 3 -c 1 -o gpurun_out/prof_r2c/spmm_c5 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/prof_r2c/ncu_spmm_c5.log 2>&1
ncu -i gpurun_out/prof_r2c/spmm_c5.ncu-rep --page raw --csv > gpurun_out/prof_r2c/spmm_c5_raw.csv 2>/dev/null
ls gpurun_out/prof_r2c
