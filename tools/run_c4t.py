"""c4t (NEXT-4) full-size solve on the GPU: per-window iterations, time, Krylov steps, and the
distance to the c4 golden fixed point (same physics, scalar J̄)."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
from _helpers import to_dev
from workloads import config, make_u0
import paper_2304_14021_b200 as pd
name = sys.argv[1] if len(sys.argv) > 1 else "c4t"
p = config(name)
u0 = make_u0(p)
s = pd.Solver(p)
U = s.empty()
prof_on = os.environ.get("C4T_PROFILE", "1") == "1"   # profiling keeps the host Arnoldi loop
s.profile(prof_on)
torch.cuda.synchronize(); t = time.time()
rc, info = s.solve(to_dev(u0), U)
torch.cuda.synchronize(); dt = time.time() - t
prof = s.profile_read() if prof_on else {}
print(name, "rc", rc, "iters", list(info.iters[:p.n_windows]), "seconds", round(dt, 3))
for k, (n, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:22s} {n:6d} {ms:9.2f} ms")
g = json.load(open(os.path.join(ROOT, "tests", "golden", "c4_full.json")))
w = g["windows"][-1]
pts = [tuple(x) for x in w["points"]]
got = np.array([float(U[a, b, c]) for a, b, c in pts])
print("golden c4 iters", [x["iters"] for x in g["windows"]],
      "max |U - c4 golden| / umax", np.abs(got - np.array(w["values"])).max() / float(U.abs().max()))
