# ncu --set full of the C3 SpMM (one launch) + key throughput metrics
out=gpurun_out/prof_spmm; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_csr -s 2 -c 1 \
  -o $out/spmm_c3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-graph > $out/ncu.log 2>&1
ncu -i $out/spmm_c3.ncu-rep --page raw --csv > $out/spmm_c3_raw.csv 2>/dev/null
ncu -i $out/spmm_c3.ncu-rep --page details --csv > $out/spmm_c3_details.csv 2>/dev/null
ncu -i $out/spmm_c3.ncu-rep --page source --csv > $out/spmm_c3_source.csv 2>/dev/null
ls -la $out
