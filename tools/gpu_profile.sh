# ncu evidence for the bench workload (run under gpurun on one B200).
# usage: bash tools/gpu_profile.sh <tag> [kernel regex ...]
tag=$1; shift
out=gpurun_out/prof_$tag; mkdir -p $out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graph > $out/bench_under_ncu.log 2>&1
python tools/ncu_summary.py $out/launches.csv > $out/launches_summary.txt 2>&1
for k in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 \
    -o $out/$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph > $out/ncu_$k.log 2>&1
  ncu -i $out/$k.ncu-rep --page raw --csv > $out/${k}_raw.csv 2>/dev/null
  ncu -i $out/$k.ncu-rep --page details --csv > $out/${k}_details.csv 2>/dev/null
done
ls -la $out
