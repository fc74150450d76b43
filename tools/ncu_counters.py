"""profiles/ncu_counters.json from an `ncu --set full` capture of the c5 bench (one launch of each
hot kernel): per library kernel name, DRAM bytes per launch (roofline.traffic), the FP64-pipe
utilisation and the ncu duration.  bench.py reads it for the roofline object.

  python tools/ncu_counters.py gpurun_out/<tag>.ncu-rep [profiles/ncu_counters.json]
"""
import csv
import io
import json
import subprocess
import sys

# ncu kernel name (prefix) -> library kernel name; k_rows3 runs twice per iteration (forward, inverse)
MAP = [("k_residual_tile", "residual"), ("k_cols_cm<1, 32, 8, 0", "dtt_y_fwd"), ("k_cols_cm<1, 32, 8, 1", "dtt_y_inv"),
       ("k_cols_tma_inv", "dtt_y_inv"),
       ("k_time2d_v4", "time_solve_2d"), ("k_update", "update"), ("k_rows3", ("dtt_x_fwd", "dtt_x_inv")),
       ("k_cols3", ("dtt_y_fwd", "dtt_y_inv")), ("k_time2d_v2", "time_solve_2d")]
KEYS = {"dram__bytes_read.sum": "read", "dram__bytes_write.sum": "write", "gpu__time_duration.sum": "duration",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_cycles_pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct"}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-6, "usecond": 1e-3,
         "msecond": 1.0, "second": 1e3}


def main(path, out):
    if path.endswith(".csv"):          # the raw page already exported on the GPU box (large reports stay there)
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    res, seen = {}, {}
    for r in rows[2:]:
        kname = r[ki]
        name = None
        for pre, lib in MAP:
            if kname.startswith("void pd::" + pre) or kname.startswith(pre) or ("pd::" + pre) in kname or pre in kname:
                if isinstance(lib, tuple):
                    c = seen.get(pre, 0)
                    seen[pre] = c + 1
                    name = lib[c % 2]
                else:
                    name = lib
                break
        if not name or name in res:
            continue
        d = {"ncu_kernel": kname[:120]}
        for k, short in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if short in ("read", "write"):
                    v *= SCALE.get(u, 1.0)
                elif short == "duration":
                    v *= SCALE.get(u, 1.0)
                d[short] = v
        if "read" in d and "write" in d:
            d["traffic"] = d["read"] + d["write"]
        res[name] = d
    with open(out, "w") as f:
        json.dump({"source": path.split("/")[-1], "kernels": res}, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_counters.json")
