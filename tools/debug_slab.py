import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from test_dist_gloo import CpuOps
from paper_2304_14021_b200 import dist
from oracle import iterate
from workloads import twin, make_u0
for name, p in [("c3", twin("c3", m=128, nt=32)), ("c5", twin("c5", m=128, nt=32))]:
    P = 2
    L = dist.SlabLayout(p.n, p.nt, P)
    u0 = make_u0(p); U0 = iterate.initial_iterate(p, u0) + 0.01 * np.random.default_rng(1).uniform(-1, 1, (p.nt, p.n, p.n))
    for r in range(P):
        y0, nyl = L.rows[r]; x0, nxl = L.cols[r]
        g = dist.GpuOps(p, 0, None, y0, nyl, x0, nxl); c = CpuOps(p, y0, nyl, x0, nxl)
        U_l = np.ascontiguousarray(U0[:, y0:y0+nyl]).reshape(-1); u0_l = np.ascontiguousarray(u0[y0:y0+nyl])
        hlo = np.ascontiguousarray(U0[:, y0-2:y0]).reshape(-1) if r > 0 else None
        hhi = np.ascontiguousarray(U0[:, y0+nyl:y0+nyl+2]).reshape(-1) if r < P-1 else None
        T = lambda a: None if a is None else torch.from_numpy(a).cuda()
        rg = torch.empty(L.row_slab(r), dtype=torch.float64, device='cuda'); rc = torch.zeros(L.row_slab(r), dtype=torch.float64)
        g.residual(T(u0_l), T(U_l), T(hlo), T(hhi), rg)
        c.residual(torch.from_numpy(u0_l), torch.from_numpy(U_l), None if hlo is None else torch.from_numpy(hlo), None if hhi is None else torch.from_numpy(hhi), rc)
        e = np.abs(rg.cpu().numpy() - rc.numpy()).max() / np.abs(rc.numpy()).max(); print(name, r, "residual", e)
        xg = torch.empty_like(rg); g.xpass(rg, xg); xc = torch.zeros_like(rc); c.xpass(rc, xc)
        print(name, r, "xpass", np.abs(xg.cpu().numpy() - xc.numpy()).max() / np.abs(xc.numpy()).max())
        cols = np.random.default_rng(2).uniform(-1, 1, L.col_slab(r))
        cg = torch.from_numpy(cols.copy()).cuda(); g.ypass(cg); cc = torch.from_numpy(cols.copy()); c.ypass(cc)
        print(name, r, "ypass", np.abs(cg.cpu().numpy() - cc.numpy()).max() / np.abs(cc.numpy()).max())
        g.close()
