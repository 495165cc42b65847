# ncu --set full of the fused EvolveGCN readout at C3
mkdir -p gpurun_out/prof_r2k_c3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:readout_f16 -s 1 -c 1 \
  -o gpurun_out/prof_r2k_c3/readout_f16 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/prof_r2k_c3/ncu.log 2>&1
ncu -i gpurun_out/prof_r2k_c3/readout_f16.ncu-rep --page raw --csv > gpurun_out/prof_r2k_c3/readout_f16_raw.csv 2>/dev/null
tail -3 gpurun_out/prof_r2k_c3/ncu.log; ls -la gpurun_out/prof_r2k_c3
