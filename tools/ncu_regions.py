"""Per-region stall breakdown of one kernel's SASS from an .ncu-rep (source page, sass view).
usage: python tools/ncu_regions.py REP KERNEL_REGEX [instructions_per_region]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
seg = int(sys.argv[3]) if len(sys.argv) > 3 else 150
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kre,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
si, st, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
sc = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


tot = sum(num(r[st]) for r in data) or 1
print("instructions", len(data), "samples", tot, "executed", sum(num(r[ie]) for r in data))
for i in range(0, len(data), seg):
    chunk = data[i:i + seg]
    s = sum(num(r[st]) for r in chunk)
    ex = sum(num(r[ie]) for r in chunk)
    reasons = {}
    ops = {}
    for r in chunk:
        for c in sc:
            v = num(r[c])
            if v:
                reasons[h[c][6:]] = reasons.get(h[c][6:], 0) + v
        t = r[si].split()
        op = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "?")).split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    top = ", ".join(f"{k}={100 * v / tot:.1f}" for k, v in sorted(reasons.items(), key=lambda x: -x[1])[:4])
    topops = ",".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:5])
    print(f"{i:5d} {100 * s / tot:5.1f}% exec {ex / 1e6:9.1f}M | {top} | {topops}")
