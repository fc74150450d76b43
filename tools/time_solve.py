"""Wall time of paradiag_solve for a config with the device-side loop (graph) and the host loop."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
from _helpers import to_dev
from workloads import config, make_u0
import paper_2304_14021_b200 as pd
for name in sys.argv[1:]:
    p = config(name)
    u0 = to_dev(make_u0(p))
    for g in ("1", "0"):
        os.environ["PARADIAG_GRAPH"] = g
        s = pd.Solver(p)
        U = s.empty()
        s.solve(u0, U)                      # warm (captures the graph)
        torch.cuda.synchronize()
        t = time.perf_counter()
        reps = 5
        for _ in range(reps):
            rc, info = s.solve(u0, U)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / reps
        it = sum(info.iters[:p.n_windows])
        print(f"{name} graph={g}: {dt*1e3:.2f} ms per solve, {it} iterations, {dt/it*1e6:.1f} us/iteration")
        s.close()
