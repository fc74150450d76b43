"""Time-slab vs single-handle statistics on one GPU: prints ‖δ‖∞ / ‖U‖∞ of both and max|ΔU|."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ["PARADIAG_TLONG"] = "1"
import torch
from _helpers import to_dev
from oracle import iterate
from workloads import twin, make_u0
import paper_2304_14021_b200 as pd
from paper_2304_14021_b200 import dist
for theta in (1.0, 0.5):
    p = twin("c6", m=32, nt=2048, t_window=2048 / 2.0 ** 20, theta=theta)
    u0 = make_u0(p).reshape(-1)
    U0 = iterate.initial_iterate(p, u0)
    s = pd.Solver(p)
    U = to_dev(U0, p); u0d = to_dev(u0)
    rk = dist.TimeSlabRank(dist.TslabOps(p, 0), 0, 1)
    Uv = U.reshape(-1).clone()
    info = None
    for k in range(3):
        prev = U.clone()
        info = s.iterate(u0d, U, info)
        st = dist.iterate_tslab_virtual([rk], u0d, [Uv])
        torch.cuda.synchronize()
        print(theta, k, "single", info.delta_max, info.u_max, "tslab", st, "true", float((U - prev).abs().max()), float(U.abs().max()),
              "eq", bool(torch.equal(U.reshape(-1), Uv)))
