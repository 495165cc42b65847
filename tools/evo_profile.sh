# ncu --set full of the EvolveGCN weight-evolution kernels on C3 (one launch each)
out=gpurun_out/prof_evo; mkdir -p $out
for k in evolve_fwd_rr evolve_bwd_rr; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 \
    -o $out/$k python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-graph > $out/ncu_$k.log 2>&1
  ncu -i $out/$k.ncu-rep --page raw --csv > $out/${k}_raw.csv 2>/dev/null
  ncu -i $out/$k.ncu-rep --page details --csv > $out/${k}_details.csv 2>/dev/null
done
ls -la $out
