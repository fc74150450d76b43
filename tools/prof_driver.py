"""Small driver for ncu: a few ParaDiag iterations of a c5-shaped problem (full 2049² grid,
reduced N_t) through the public C ABI.  usage: python tools/prof_driver.py [nt] [iters] [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace  # noqa: E402

import torch  # noqa: E402

import paper_2304_14021_b200 as pd  # noqa: E402
from workloads import config, make_u0  # noqa: E402

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 16
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
name = sys.argv[3] if len(sys.argv) > 3 else "c5"
m = int(sys.argv[4]) if len(sys.argv) > 4 else config(name).m
p = replace(config(name), nt=nt, m=m, t_window=config(name).t_window * nt / config(name).nt)
s = pd.Solver(p)
u0 = torch.from_numpy(make_u0(p)).cuda()
U = torch.zeros(s.shape, dtype=torch.float64, device="cuda")
info = None
for _ in range(iters):
    info = s.iterate(u0, U, info)
torch.cuda.synchronize()
print("ok", info.delta_max, info.u_max)
