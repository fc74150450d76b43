"""the oracle (as it stands) timed on the host cores of the GPU box, per config,
with 1 BLAS thread and with all of them.  A reported CPU baseline, not the target.

  python tools/cpu_baseline.py [out.json]

Per config: one warm-up iteration then the median of `reps` iterations of oracle.iterate.iterate_once
(residual, naive O(N_t²) DFT, Step-(2) solves, inverse DFT, update) on the config's own grid, except
c5 (17 GB per array; the oracle would need > 50 GB and minutes per iteration), which runs on the
bounded 65² x N_t = 512 twin bench.py's cpu_baseline uses — said in the row.  dof/s = dofs / s.
"""
import json
import os
import platform
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

from oracle import iterate  # noqa: E402
from workloads import config, twin, make_u0  # noqa: E402


def cpu_info():
    info = {"machine": platform.machine(), "logical_cpus": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k.strip()] = v.strip()
    except Exception:
        pass
    try:
        with open("/proc/meminfo") as f:
            info["MemTotal"] = f.readline().split(":")[1].strip()
    except Exception:
        pass
    return info


def time_config(name, threads, reps):
    p = config(name)
    sample = "full config"
    if name == "c5":
        p = twin("c5", m=64)
        sample = "65^2 x N_t=512 twin (full c5 needs > 50 GB in the oracle)"
    u0 = make_u0(p)
    if p.dim == 1:
        u0 = u0.reshape(-1)
    U = iterate.initial_iterate(p, u0)
    with threadpool_limits(limits=threads):
        U, _ = iterate.iterate_once(p, u0, U)         # warm-up
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            U, _ = iterate.iterate_once(p, u0, U)
            ts.append(time.perf_counter() - t0)
    s = statistics.median(ts)
    return {"config": name, "threads": threads, "dofs": p.dofs, "s_per_iteration": s, "dof_per_s": p.dofs / s,
            "reps": reps, "sample": sample}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "cpu_baseline.json")
    allc = os.cpu_count()
    rows = []
    for name, reps in (("c1", 5), ("c2", 3), ("c3", 1), ("c4", 2), ("c5", 1)):
        for th in (1, allc):
            r = time_config(name, th, reps)
            rows.append(r)
            print(json.dumps(r), flush=True)
    res = {"cpu": cpu_info(), "numpy": np.__version__, "rows": rows,
           "what": "oracle.iterate.iterate_once (numpy fp64, naive O(N_t^2) DFT, dense DCT/DST matmuls, banded LU "
                   "+ refinement in 1D), median of reps after one warm-up; BLAS threads limited per row"}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
