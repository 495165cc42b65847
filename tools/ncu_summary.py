"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel shares: python tools/ncu_summary.py launches.csv"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"(\(anonymous namespace\)|<unnamed>)::", "", name)
    name = re.sub(r"^void ", "", name)
    m = re.match(r"([\w:]+)", name)
    return m.group(1) if m else name


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        a = agg[short(r[ki])]
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':36s} {'launches':>8s} {'total us':>10s} {'mean us':>9s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:36s} {n:8d} {t / 1e3:10.1f} {t / n / 1e3:9.1f} {t / tot * 100:5.1f}%")
    print(f"{'TOTAL':36s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
