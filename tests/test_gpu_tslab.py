"""Time slabs on ONE GPU (1D long windows across ranks; dist.TimeSlabRank):
P virtual ranks run the phases in rank order with the halo row and the two all-to-alls emulated by
copies (dist.iterate_tslab_virtual), each rank with its own handle of the global problem, against
the unsharded long-window iteration of one handle (paradiag_iterate, itself pinned to the oracle
in tests/test_gpu_tlong.py) and, at oracle sizes, against the oracle.

Every time pencil goes through the same kernels with the same pairing (2p, 2p+1) of spatial modes,
the halo row is the same value the unsharded residual reads, and the norms are maxima, so the
sharded iterates equal the unsharded ones bit for bit.  A one-rank NCCL world runs the real
collectives (TorchComm) through the same path."""
import numpy as np
import pytest

from _helpers import to_dev, rel_err, oracle_u0
from oracle import iterate
from workloads import twin, make_u0

pytestmark = pytest.mark.gpu


def _c6(nt, m=64, **kw):
    """c6 physics (hinged biharmonic, Δt = 2^-20) at a shorter window."""
    return twin("c6", m=m, nt=nt, t_window=nt / 2.0 ** 20, **kw)


FORCED = {                                     # PARADIAG_TLONG=1: the four-step path from N_t = 1024
    "c6_nt1024": _c6(1024),                    # N_x = 63, pitch 64
    "c6_m32_nt2048_theta": _c6(2048, m=32, theta=0.5),   # N_x = 31, pitch 32
}
UNFORCED = {
    "c6_nt8192": _c6(8192),                    # five-stage time pass (N2 = 64)
    "c6_nt32768": _c6(32768),                  # fused pass B (N2 = 1024)
}
# c6n physics (Neumann, 65 nodes: DMMA x path with the x-mode pitch 80, so 2, 4, 8 ranks get even
# column blocks) with a mixed-radix window (2000 = 40 x 50, k_tmix.cuh)
MIXED = {"c6n_nt2000": twin("c6n", nt=2000, t_window=2000e-6)}
CASES = {**FORCED, **UNFORCED, **MIXED}


def _run(cuda_lib, monkeypatch, name, P, K=3):
    import torch
    from paper_2304_14021_b200 import dist
    if name in FORCED:
        monkeypatch.setenv("PARADIAG_TLONG", "1")
    p = CASES[name]
    u0 = make_u0(p).reshape(-1)
    U0 = iterate.initial_iterate(p, u0)
    s = cuda_lib.Solver(p)
    U = to_dev(U0, p)
    u0d = to_dev(u0)
    ranks = [dist.TimeSlabRank(dist.TslabOps(p, 0), r, P) for r in range(P)]
    nn = ranks[0].nn
    Us = [U.reshape(p.nt, -1)[r * nn:(r + 1) * nn].clone().reshape(-1) for r in range(P)]   # never alias U
    out = []
    info = None
    for _ in range(K):
        info = s.iterate(u0d, U, info)
        st = dist.iterate_tslab_virtual(ranks, u0d, Us)
        torch.cuda.synchronize()
        got = torch.cat([x.reshape(nn, -1) for x in Us], dim=0)
        out.append((got.cpu().numpy(), U.reshape(p.nt, -1).cpu().numpy(), st, (info.delta_max, info.u_max)))
    for rk in ranks:
        rk.ops.close()
    s.close()
    return p, u0, U0, out


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("name", sorted(CASES))
def test_virtual_time_slabs_match_single_gpu(cuda_lib, monkeypatch, name, P):
    p, u0, U0, out = _run(cuda_lib, monkeypatch, name, P)
    for got, ref, st, st_ref in out:
        assert np.array_equal(got, ref), rel_err(got, ref)
        assert st == st_ref


@pytest.mark.parametrize("name", sorted(FORCED) + sorted(MIXED))
def test_virtual_time_slabs_match_oracle(cuda_lib, monkeypatch, name):
    p, u0, U0, out = _run(cuda_lib, monkeypatch, name, 4, K=2)
    U_o = U0
    for got, _, st, _ in out:
        U_o, info = iterate.iterate_once(p, oracle_u0(p, u0), U_o)
        assert rel_err(got, U_o) <= 1e-10
        assert abs(st[0] - info["delta_max"]) <= 1e-10 * info["u_max"]


def test_time_slab_entry_points_reject_bad_arguments(cuda_lib, monkeypatch):
    import torch
    import paper_2304_14021_b200 as pd
    monkeypatch.setenv("PARADIAG_TLONG", "1")
    p = FORCED["c6_nt1024"]
    s = cuda_lib.Solver(p)
    h = s.h
    assert pd.paradiag_tslab_pitch(h) == 64
    U = torch.zeros(8 * 63, dtype=torch.float64, device="cuda")
    row = torch.zeros(63, dtype=torch.float64, device="cuda")
    blocks = torch.zeros(64 * 8, dtype=torch.float64, device="cuda")
    cols = torch.zeros(1024 * 16, dtype=torch.float64, device="cuda")
    for bc in (0, 3, 6, 128):                  # zero, odd, not dividing the pitch, too wide
        with pytest.raises(pd.ParadiagError):
            pd.paradiag_tslab_residual(h, row, U, 8, blocks, bc)
    with pytest.raises(pd.ParadiagError):
        pd.paradiag_tslab_residual(h, row, U, 0, blocks, 8)          # no rows
    with pytest.raises(pd.ParadiagError):
        pd.paradiag_tslab_time(h, cols, 8, 16)                       # c0 not a block start
    with pytest.raises(pd.ParadiagError):
        pd.paradiag_tslab_time(h, cols, 64, 16)                      # past the pitch
    with pytest.raises(pd.ParadiagError):
        pd.paradiag_tslab_update(h, blocks, 8, U, 1 << 20)           # more rows than N_t
    s.close()
    q = cuda_lib.Solver(twin("c5", m=16, nt=8))                       # 2D handle: not a time-slab handle
    with pytest.raises(pd.ParadiagError):
        pd.paradiag_tslab_time(q.h, cols, 0, 16)
    q.close()


def _nccl_world1(out_q):
    import os
    import socket
    import torch
    import torch.distributed as tdist
    from paper_2304_14021_b200 import dist
    import paper_2304_14021_b200 as pd
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    try:
        p = UNFORCED["c6_nt8192"]
        u0 = make_u0(p).reshape(-1)
        U0 = iterate.initial_iterate(p, u0)
        stream = torch.cuda.current_stream()
        rk = dist.TimeSlabRank(dist.TslabOps(p, 0, stream.cuda_stream), 0, 1)
        comm = dist.TorchComm()
        U = to_dev(U0, p).reshape(-1).clone()
        u0d = to_dev(u0)
        s = pd.Solver(p)
        Ur = to_dev(U0, p)
        info = None
        errs = []
        for _ in range(3):
            rk.iterate(u0d, U, comm)
            info = s.iterate(u0d, Ur, info)
            errs.append(rel_err(U.reshape(Ur.shape).cpu().numpy(), Ur.cpu().numpy()))
        rk.ops.close()
        out_q.put(errs)
    finally:
        tdist.destroy_process_group()


def test_nccl_time_slabs_world1(cuda_lib):
    """The real NCCL all-to-alls, halo exchange and max all-reduce of TimeSlabRank.iterate in a
    one-rank world (one process, one device) against the unsharded iteration."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_nccl_world1, args=(q,))
    pr.start()
    errs = q.get(timeout=600)
    pr.join(timeout=600)
    assert pr.exitcode == 0
    assert max(errs) == 0.0, errs
