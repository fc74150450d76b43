"""Summarise an .ncu-rep: key throughput/occupancy/stall metrics per kernel (run here, no GPU)."""
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sector_hit_rate.pct"]
STALL = re.compile(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active.ratio")


def main(path):
    if path.endswith(".csv"):          # the raw page already exported on the GPU box (large reports stay there)
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    for r in rows[2:]:
        print("=====", r[ki][:90])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {r[i]:>16s} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            m = STALL.match(h)
            if m and r[i]:
                try:
                    stalls.append((float(r[i]), m.group(1)))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("  top stalls:", ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
