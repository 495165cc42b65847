out=gpurun_out/prof_evo; mkdir -p $out
for cl in; do
  echo "== DGC_EVOLVE_CL=$cl"
  DGC_EVOLVE_CL=$cl timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --detail > gpurun_out/evo_cl$cl.log 2>&1
  grep -E "^evolve" gpurun_out/evo_cl$cl.log; grep -o '"epoch_ms": [0-9.]*' gpurun_out/evo_cl$cl.log
done
for k in evolve_fwd_cl evolve_bwd_cl; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 \
    -o $out/$k python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-graph > $out/ncu_$k.log 2>&1
  ncu -i $out/$k.ncu-rep --page raw --csv > $out/${k}_raw.csv 2>/dev/null
  ncu -i $out/$k.ncu-rep --page details --csv > $out/${k}_details.csv 2>/dev/null
  ncu -i $out/$k.ncu-rep --page source --csv > $out/${k}_source.csv 2>/dev/null
done
ls -la $out
