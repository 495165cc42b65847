python tools/time_gemm_c2.py
mkdir -p gpurun_out/prof_gemm
for w in stacked dh2; do
timeout 600 ncu --set full --clock-control none -k regex:gemm_tf32 -s 1 -c 1 -o gpurun_out/prof_gemm/$w python tools/time_gemm_c2.py $w > /dev/null 2>&1
ncu -i gpurun_out/prof_gemm/$w.ncu-rep --page raw --csv > gpurun_out/prof_gemm/${w}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_gemm/$w.ncu-rep --page details --csv > gpurun_out/prof_gemm/${w}_details.csv 2>/dev/null
done
