"""Top SASS instructions by stall samples, and instruction-class totals, from an .ncu-rep."""
import collections
import csv
import io
import subprocess
import sys

path = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"] +
                     (["-k", kfilter] if kfilter else []), capture_output=True, text=True).stdout
lines = out.splitlines()
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
for b in blocks:
    name = b[0].split(",")[1][:80]
    rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
    h = rows[0]
    si, ii, ti = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = []
    cls = collections.Counter()
    stall_cls = collections.Counter()
    for r in rows[1:]:
        try:
            s = int(r[ii] or 0)
            n = int(r[ti] or 0)
        except ValueError:
            continue
        op = r[si].strip().split()[0] if r[si].strip() else "?"
        if op.startswith("@"):
            op = r[si].strip().split()[1]
        base = op.split(".")[0]
        cls[base] += n
        stall_cls[base] += s
        data.append((s, r[si].strip()[:70], n))
    tot = sum(x[0] for x in data) or 1
    print("=====", name, "samples", tot)
    for s, src, n in sorted(data, reverse=True)[:25]:
        print(f"  {100*s/tot:5.1f}%  {n:>10d}  {src}")
    print("  instr classes (executed):", ", ".join(f"{k}={v}" for k, v in cls.most_common(14)))
    print("  stall by class:", ", ".join(f"{k}={100*v/tot:.0f}%" for k, v in stall_cls.most_common(10)))
