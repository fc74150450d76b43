"""Time slabs (1D long windows across ranks; dist.TimeSlabRank) on CPU.

The orchestration of paper_2304_14021_b200/dist.py — contiguous time rows per rank for the residual
and the x transforms, the halo row, the two all-to-alls into x-mode column blocks of all N_t rows
and back, the max-reductions — runs with a CPU stand-in for the library's paradiag_tslab_* calls
built from the oracle's pieces (this file), against the oracle's unsharded iteration:
  * all P ranks in one process (dist.iterate_tslab_virtual, P = 1, 2, 4);
  * world size 2 over torch.distributed gloo (real collectives, TorchComm).
The GPU path (tests/test_gpu_tslab.py) runs the same classes with the real kernels."""
import os
import socket
from dataclasses import replace

import numpy as np
import pytest
import torch

from oracle import circulant, iterate, spatial, precond
from workloads import twin, make_u0


def _case(nt, m=16, **kw):
    """c6 physics (hinged biharmonic, Δt = 2^-20) on a short window and a small grid."""
    return twin("c6", m=m, nt=nt, t_window=nt / 2.0 ** 20, **kw)


CASES = {"c6_m16_nt16": _case(16), "c6_m32_nt32_theta": _case(32, m=32, theta=0.5)}


class TslabCpuOps:
    """CPU stand-in for dist.TslabOps: the same layouts and conventions (unnormalised x transform
    T on the rows, the time pass carries Γ_α, the per-mode divide, 1/N_t and the 1/(2m) of T⁻¹)."""

    def __init__(self, p):
        self.p = p
        self.nt = p.nt
        self.nx = spatial.n_unknowns(p.m, p.bc)
        self.pitch = 2 * ((self.nx + 1) // 2)
        self.T = spatial.transform_matrix(p.m, p.bc)
        self.dmax = self.umax = 0.0

    def empty(self, count):
        return torch.zeros(count, dtype=torch.float64)

    def residual(self, u_prev, U_l, nn, blocks, bc):
        p = self.p
        sub = replace(p, nt=nn, t_window=p.t_window * nn / p.nt)        # same Δt
        U = U_l.numpy().reshape(nn, self.nx)
        r = iterate.residual_linear(sub, u_prev.numpy().reshape(self.nx), U)
        hat = np.zeros((nn, self.pitch))
        hat[:, :self.nx] = r @ self.T.T
        b = blocks.numpy().reshape(self.pitch // bc, nn, bc)
        for q in range(self.pitch // bc):
            b[q] = hat[:, q * bc:(q + 1) * bc]

    def time(self, cols, c0, bc):
        p = self.p
        c = cols.numpy().reshape(self.nt, bc)
        ncol = min(bc, self.nx - c0)
        if ncol <= 0:
            return
        S = circulant.step1(c[:, :ncol].copy(), p.alpha)
        d = circulant.eig_d(self.nt, p.alpha, circulant.inv_dt(p))
        e = circulant.eig_e(self.nt, p.alpha, p.theta)
        mu = precond._step2_mu(p, 0.0)[c0:c0 + ncol]
        S = S / (d[:, None] + e[:, None] * mu[None, :])
        x, _ = circulant.step3(S, p.alpha)
        c[:, :ncol] = x / (2.0 * p.m)

    def update(self, blocks, bc, U_l, nn):
        b = blocks.numpy().reshape(self.pitch // bc, nn, bc)
        hat = np.concatenate(list(b), axis=1)[:, :self.nx]
        delta = hat @ self.T.T
        U = U_l.numpy().reshape(nn, self.nx)
        U += delta
        self.dmax = max(self.dmax, float(np.abs(delta).max()))
        self.umax = max(self.umax, float(np.abs(U).max()))

    def stats_reset(self):
        self.dmax = self.umax = 0.0

    def stats_read(self):
        return self.dmax, self.umax


def _oracle_iterates(p, u0, K):
    U = iterate.initial_iterate(p, u0)
    out = []
    for _ in range(K):
        U, info = iterate.iterate_once(p, u0, U)
        out.append((U.copy(), info))
    return out


def _check(p, got, stats, ref):
    for k, (U, info) in enumerate(ref):
        assert abs(stats[k][0] - info["delta_max"]) <= 1e-11 * max(info["u_max"], info["delta_max"])
        assert abs(stats[k][1] - info["u_max"]) <= 1e-11 * info["u_max"]
    U = ref[-1][0]
    assert np.abs(got - U).max() <= 1e-11 * np.abs(U).max()


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("name", sorted(CASES))
def test_virtual_time_slabs_match_oracle(name, P):
    from paper_2304_14021_b200 import dist
    p = CASES[name]
    u0 = make_u0(p).reshape(-1)
    U0 = iterate.initial_iterate(p, u0)
    ranks = [dist.TimeSlabRank(TslabCpuOps(p), r, P) for r in range(P)]
    nn = ranks[0].nn
    Us = [torch.from_numpy(np.ascontiguousarray(U0[r * nn:(r + 1) * nn]).reshape(-1)) for r in range(P)]
    u0t = torch.from_numpy(u0.copy())
    K = 3
    stats = [dist.iterate_tslab_virtual(ranks, u0t, Us) for _ in range(K)]
    got = np.concatenate([U.numpy().reshape(nn, -1) for U in Us], axis=0)
    _check(p, got, stats, _oracle_iterates(p, u0, K))


def test_time_slab_geometry():
    from paper_2304_14021_b200 import dist
    assert dist.tslab_geometry(1 << 20, 64, 8) == (1 << 17, 8)
    assert dist.tslab_geometry(16, 16, 2) == (8, 8)
    for bad in [(16, 16, 3), (16, 18, 2), (16, 16, 16), (8, 64, 16)]:
        with pytest.raises(ValueError):
            dist.tslab_geometry(*bad)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, K, out):
    import torch.distributed as tdist
    from paper_2304_14021_b200 import dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = CASES[name]
        u0 = make_u0(p).reshape(-1)
        U0 = iterate.initial_iterate(p, u0)
        rk = dist.TimeSlabRank(TslabCpuOps(p), rank, world)
        nn = rk.nn
        U_l = torch.from_numpy(np.ascontiguousarray(U0[rank * nn:(rank + 1) * nn]).reshape(-1))
        comm = dist.TorchComm()
        stats = [rk.iterate(torch.from_numpy(u0.copy()), U_l, comm) for _ in range(K)]
        gathered = [torch.zeros_like(U_l) for _ in range(world)]
        tdist.all_gather(gathered, U_l)
        if rank == 0:
            np.save(out, np.concatenate([g.numpy().reshape(nn, -1) for g in gathered], axis=0))
            np.save(out + ".stats.npy", np.array(stats))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("name", sorted(CASES))
def test_two_rank_gloo_time_slabs_match_oracle(tmp_path, name):
    import torch.multiprocessing as mp
    p = CASES[name]
    K = 2
    out = str(tmp_path / "U.npy")
    mp.spawn(_worker, args=(2, _free_port(), name, K, out), nprocs=2, join=True)
    _check(p, np.load(out), np.load(out + ".stats.npy"), _oracle_iterates(p, make_u0(p).reshape(-1), K))
