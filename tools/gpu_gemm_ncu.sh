# per-launch metrics of every GEMM launch in one eager C2 epoch (names carry the template args)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,launch__grid_size \
  -k regex:gemm_tf32_kernel --launch-skip 40 --launch-count 20 --clock-control none --csv --log-file gpurun_out/gemm_ncu.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/gemm_ncu.out 2> gpurun_out/gemm_ncu.err
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/gemm_ncu.csv")) if len(r) > 10]
hdr = rows[0]; ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault(r[ii], {"name": r[ki][:70]})[r[mi]] = r[vi]
for k, v in d.items():
    print(v["name"], "|", v.get("gpu__time_duration.sum"), "us | rd", v.get("dram__bytes_read.sum"), "wr", v.get("dram__bytes_write.sum"),
          "| sm%", v.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"), "lts%", v.get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
          "| lsb", v.get("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"), "grid", v.get("launch__grid_size"))
PY
