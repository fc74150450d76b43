import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from test_dist_gloo import CpuOps
from paper_2304_14021_b200 import dist
from oracle import iterate
from workloads import twin, make_u0
p = twin("c3", m=128, nt=32); P = 2
L = dist.SlabLayout(p.n, p.nt, P)
u0 = make_u0(p); U0 = iterate.initial_iterate(p, u0)
gr, cr = [], []
for r in range(P):
    y0, nyl = L.rows[r]; x0, nxl = L.cols[r]
    gr.append(dist.SlabRank(L, r, dist.GpuOps(p, 0, None, y0, nyl, x0, nxl)))
    cr.append(dist.SlabRank(L, r, CpuOps(p, y0, nyl, x0, nxl)))
Ug = [torch.from_numpy(np.ascontiguousarray(U0[:, y0:y0+n]).reshape(-1)).cuda() for y0, n in L.rows]
Uc = [torch.from_numpy(np.ascontiguousarray(U0[:, y0:y0+n]).reshape(-1)) for y0, n in L.rows]
u0g = [torch.from_numpy(np.ascontiguousarray(u0[y0:y0+n])).cuda() for y0, n in L.rows]
u0c = [torch.from_numpy(np.ascontiguousarray(u0[y0:y0+n])) for y0, n in L.rows]
def cmp(tag, a, b):
    a = a.cpu().numpy(); b = b.numpy(); print(tag, np.abs(a-b).max() / max(np.abs(b).max(), 1e-300), np.abs(b).max())
for rs, Us, us in ((gr, Ug, u0g), (cr, Uc, u0c)):
    for k in range(P): rs[k].phase_halo_pack(Us[k])
    for k in range(P):
        if k > 0: rs[k].hlo.copy_(rs[k-1].hsend_hi)
        if k < P-1: rs[k].hhi.copy_(rs[k+1].hsend_lo)
for k in range(P):
    for nm in ("hsend_lo", "hsend_hi"): cmp(f"r{k} {nm}", getattr(gr[k], nm), getattr(cr[k], nm))
for rs, Us, us in ((gr, Ug, u0g), (cr, Uc, u0c)):
    for k in range(P):
        rs[k].ops.residual(us[k], Us[k], rs[k].hlo, rs[k].hhi, rs[k].rows)
for k in range(P): cmp(f"r{k} residual", gr[k].rows, cr[k].rows)
for rs in (gr, cr):
    for k in range(P):
        rs[k].ops.xpass(rs[k].rows, rs[k].rows)
        for d in L.fwd_pack(k): rs[k].ops.copy(rs[k].rows, rs[k].send, d)
for k in range(P): cmp(f"r{k} xfwd", gr[k].rows, cr[k].rows); cmp(f"r{k} send", gr[k].send, cr[k].send)
for rs in (gr, cr): dist._alltoall_virtual(rs, [L.fwd_send_splits(k) for k in range(P)])
for k in range(P): cmp(f"r{k} recv", gr[k].recv, cr[k].recv)
for rs in (gr, cr):
    for k in range(P): rs[k].phase_ypass()
for k in range(P): cmp(f"r{k} cols", gr[k].cols, cr[k].cols); cmp(f"r{k} send2", gr[k].send, cr[k].send)
for rs in (gr, cr): dist._alltoall_virtual(rs, [L.bwd_send_splits(k) for k in range(P)])
for rs, Us in ((gr, Ug), (cr, Uc)):
    for k in range(P): rs[k].phase_xinv_update(Us[k])
for k in range(P): cmp(f"r{k} delta", gr[k].rows, cr[k].rows); cmp(f"r{k} U", Ug[k], Uc[k])
