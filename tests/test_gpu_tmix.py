"""NEXT-3 as the paper states it: long windows with N_t = 2^a 5^b ("Δt = 10⁻⁶, i.e.
N_t = 10⁶", P:717 N_t = 10⁴), solved by the mixed-radix four-step time pass (csrc/k_tmix.cuh).

* P_α⁻¹ element-wise against the oracle (naive O(N_t²) DFT, banded LU / eigenbasis Step (2)) for
  mixed lengths whose factor transforms exercise every radix (2, 4, 5, 8) and plan shape, in 1D
  (Neumann lines: generic x passes; hinged N_x ≤ 64: the DMMA x path) and 2D.
* Solves against the oracle on reduced windows (same h and Δt as c6n).
* The full c6n window (N_t = 10⁶, Neumann, h = 1/64): iteration count and sampled iterates against
  the closed-form per-mode WR iterate (oracle/modespace.py).
Bars as test_gpu_tlong.py (1D: 1e-11 plus twice the oracle's LU-vs-eigenbasis floor)."""
from dataclasses import replace

import numpy as np
import pytest

from _helpers import gshape, to_dev, to_host, rel_err, oracle_u0, rounding_floor_1d, eigenbasis_precond_1d
from oracle import iterate, precond, modespace
from workloads import config, twin, make_u0

pytestmark = pytest.mark.gpu

DT = 1e-6


def _c6n(nt, **kw):
    return replace(config("c6n"), name="c6n_twin", nt=nt, t_window=nt * DT, **kw)


PRECOND = {
    "c6n_nt1000": _c6n(1000),                                   # 40 x 25: plans (8,5) / (5,5)
    "c6n_nt1280": _c6n(1280),                                   # 32 x 40: (8,4) / (8,5)
    "c6n_nt625": _c6n(625),                                     # odd N: 25 x 25, no Nyquist bin
    "c6n_nt2000_theta": _c6n(2000, theta=0.5),                  # 40 x 50, trapezoid e_l
    "c6n_nt10000": _c6n(10 ** 4),                               # P:717's N_t = 10^4: 100 x 100, (4,5,5)
    "c6h_nt2000": replace(config("c6"), nt=2000, t_window=2000 * DT),   # hinged 63 unknowns: DMMA x path
    "c2_nt1000": twin("c2", m=64, nt=1000, t_window=1.0),       # linear CH, Neumann growing modes
    "c5_m32_nt1000": twin("c5", m=32, nt=1000, t_window=0.5),   # 2D Neumann, mixed time pass
    "c3_m32_nt1250": twin("c3", m=32, nt=1250, t_window=0.05),  # 2D hinged, 25 x 50
}


@pytest.mark.parametrize("name", sorted(PRECOND))
def test_mixed_radix_precond_parity(cuda_lib, name):
    p = PRECOND[name]
    r = np.random.default_rng(31).uniform(-1, 1, gshape(p))
    s = cuda_lib.Solver(p)
    rd = to_dev(r, p)
    d = s.empty()
    s.apply_precond(rd, d, 0.0)
    r_o = r.reshape(p.nt, p.nx) if p.dim == 1 else r
    d_o, _ = precond.apply_precond(p, r_o, 0.0)
    bar = 1e-11 + 2 * rounding_floor_1d(p, r_o, d_o) if p.dim == 1 else 1e-11
    assert rel_err(to_host(d, p), d_o) <= bar
    if p.dim == 1:
        assert rel_err(to_host(d, p), eigenbasis_precond_1d(p, r_o)) <= bar
    s.apply_precond(rd, rd, 0.0)                                # in place
    assert rel_err(to_host(rd, p), d_o) <= bar


@pytest.mark.parametrize("name", ["c6n_nt1000", "c6n_nt2000_theta", "c6h_nt2000"])
def test_mixed_radix_solve_parity(cuda_lib, name):
    p = PRECOND[name]
    u0 = make_u0(p)
    s = cuda_lib.Solver(p)
    U = s.empty()
    rc, info = s.solve(to_dev(u0), U)
    U_o, iters_o, conv_o, _ = iterate.solve(p, oracle_u0(p, u0))
    assert list(info.iters[:1]) == iters_o and rc == 0 and all(conv_o)
    assert rel_err(to_host(U, p), U_o) <= 1e-10


def test_c6n_full_window_1e6(cuda_lib):
    """c6n: N_t = 10⁶ (Δt = 10⁻⁶), Neumann, h = 1/64.  The iteration reaches the stopping
    rule in 3 iterations from the broadcast start (the paper reports 4 from a random start against
    the sequential solution, R#4/R#5), and the iterate equals the closed-form per-mode WR iterate
    at sampled points of the whole window."""
    import torch
    p = config("c6n")
    u0 = make_u0(p)
    s = cuda_lib.Solver(p)
    U = s.empty()
    rc, info = s.solve(to_dev(u0), U)
    assert rc == 0 and info.converged
    K = info.iters[0]
    assert K == 3
    rng = np.random.default_rng(66)
    pts = [(int(rng.integers(p.nt)), 0, int(rng.integers(p.nx))) for _ in range(40)]
    pts += [(0, 0, 0), (1, 0, p.nx - 1), (p.nt // 2, 0, 32), (p.nt - 1, 0, 0), (p.nt - 1, 0, p.nx - 1)]
    idx = torch.tensor([[n, ix] for n, _, ix in pts], device=U.device)
    got = U.reshape(p.nt, p.nx)[idx[:, 0], idx[:, 1]].cpu().numpy()
    g, c0 = modespace.mode_iterates(p, u0, K)
    ref = modespace.sample(p, g, c0, pts)
    assert np.abs(got - ref).max() <= 1e-10 * float(U.abs().max())


@pytest.mark.parametrize("name", ["c6n_nt1000", "c6n_nt625", "c6n_nt2000_theta", "c5_m32_nt1000"])
def test_mixed_fused_pass_b_matches_unfused(cuda_lib, monkeypatch, name):
    """The fused mixed-radix pass B (k_mx_b_fused: forward DIF, the Hermitian-pair divide at the
    digit-reversed positions, inverse DIT, Y read and written once) against the three-kernel
    sequence (pass B, k_tl_divide, pass B⁻¹), each pinned to the oracle above: the same operations,
    so they agree to rounding (odd N1 = 25 exercises the self-mirrored k1 = 0 group alone)."""
    p = PRECOND[name]
    r = np.random.default_rng(29).uniform(-1, 1, gshape(p))
    out = []
    for fuse in ("1", "0"):
        monkeypatch.setenv("PARADIAG_TLFUSE", fuse)
        s = cuda_lib.Solver(p)
        d = s.empty()
        s.apply_precond(to_dev(r, p), d, 0.0)
        out.append(to_host(d, p))
        s.close()
    assert rel_err(out[0], out[1]) <= 1e-12
