"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv): per-kernel count, average
device time and share of the listed launches.  usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':52s} {'launches':>8s} {'avg ms':>10s} {'share':>6s}")
    for k, v in agg.items():
        print(f"{k[:52]:52s} {len(v):8d} {sum(v) / len(v) / 1e6:10.3f} {sum(v) / tot:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
