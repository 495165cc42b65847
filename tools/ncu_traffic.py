"""Build profiles/ncu_traffic.json from `ncu --set full` raw CSV exports
(tools/gpu_profile.sh, tools/evo_profile.sh): per kernel the DRAM bytes of the
captured launch, its duration and the headline utilisation metrics. bench.py
attaches `traffic` to its roofline when the record's config and shape are the
dominant kernel's.

usage: python tools/ncu_traffic.py OUT.json TAG CONFIG:BENCH_NAME:RAW_CSV[:SHAPE] ...
"""
import csv
import json
import sys


def metric(hdr, units, val, name):
    i = hdr.index(name)
    v = float(val[i].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ns": 1e-3, "ms": 1e3}
    return v * scale.get(units[i], 1)


def record(path):
    rows = list(csv.reader(open(path)))
    hdr, units, val = rows[0], rows[1], rows[2]
    rd = metric(hdr, units, val, "dram__bytes_read.sum")
    wr = metric(hdr, units, val, "dram__bytes_write.sum")
    tensor = [h for h in hdr if h.startswith("sm__pipe_tensor") and h.endswith("pct_of_peak_sustained_active")]
    stalls = sorted(((metric(hdr, units, val, h), h) for h in hdr
                     if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
                     and "not_issued" not in h), reverse=True)[:3]
    return {
        "ncu_kernel": val[hdr.index("Kernel Name")].split("(")[0].replace("void <unnamed>::", ""),
        "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
        "duration_us": metric(hdr, units, val, "gpu__time_duration.sum"),
        "dram_pct": metric(hdr, units, val, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "tensor_pipe_pct": max((metric(hdr, units, val, h) for h in tensor), default=0.0),
        "warps_active_pct": metric(hdr, units, val, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "regs": metric(hdr, units, val, "launch__registers_per_thread"),
        "grid": metric(hdr, units, val, "launch__grid_size"),
        "top_stalls": [f"{h[len('smsp__average_warps_issue_stalled_'):].split('_per_issue')[0]} {v:.2f}"
                       for v, h in stalls],
    }


def main(out, tag, specs):
    # merge: records of other kernels / configs already in OUT are kept
    try:
        kernels = json.load(open(out)).get("kernels", {})
    except (OSError, ValueError):
        kernels = {}
    for spec in specs:
        parts = spec.split(":")
        config, name, path = parts[:3]
        rec = record(path)
        rec["config"] = config
        rec["round"] = tag
        if len(parts) > 3:
            rec["shape"] = parts[3]
        kernels[f"{config}/{name}"] = rec
    json.dump({"source": "ncu --set full --clock-control none, one launch each (-s 1/2 -c 1) of "
                         f"python bench.py --config <config> --steps 1 --warmup 1 --no-cpu-baseline "
                         f"--no-graph; round state {tag}",
               "kernels": kernels}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3:])
