"""GPU parity of the long-window time pass (k_tlong.cuh).

N_t > 4096 runs the four-step time FFT over HBM (N_t = N1·N2) with Step (2) as a per-mode divide in
the DST-I/DCT-I eigenbasis (1D and 2D).  PARADIAG_TLONG=1 forces the same path from N_t = 1024, so
the oracle (naive DFT + banded LU in 1D) checks every four-step factor length (32..128)
at sizes it finishes in seconds; N_t = 8192 is the first size that takes the path unforced.  1D rows
of N_x ≤ 64 take the DMMA x transforms of k_x1d.cuh (fused with residual and update), longer rows
the register-FFT line kernels.
BJ-style bars: P_α⁻¹ ≤ 1e-11 relative, solves ≤ 1e-10 (linear) / 1e-8 (CH) with identical counts.
Full size (c6, N_t = 2^20): iteration count and sampled iterates vs the closed-form per-mode WR
iterate (oracle/modespace.py), where the physical-space oracle would need an N_t² DFT.
"""
from dataclasses import replace

import numpy as np
import pytest

from _helpers import gshape, to_dev, to_host, rel_err, oracle_u0, rounding_floor_1d, eigenbasis_precond_1d
from oracle import iterate, precond, modespace, spatial, circulant
from workloads import config, twin, make_u0

pytestmark = pytest.mark.gpu


def _c6(nt, **kw):
    """c6 physics (Δt = 2^-20) at a shorter window."""
    return twin("c6", nt=nt, t_window=nt / 2.0 ** 20, **kw)


FORCED = {
    # (N1, N2) = (32, 32), (64, 32), (64, 64), (32, 32)
    "c6_nt1024": _c6(1024),
    "c6_nt2048_theta": _c6(2048, theta=0.5),
    "c2n_m256_nt4096": twin("c2", m=256, nt=4096, t_window=1.0),          # 257 nodes: odd N_s, Neumann
    "c2n_m32_nt1024": twin("c2", m=32, nt=1024, t_window=0.25),           # 33 nodes: DMMA x transform, Neumann
    "c3_m16_nt1024": twin("c3", m=16, nt=1024, t_window=0.4),             # 2D hinged, 225 modes
    "c5_m8_nt2048_theta": twin("c5", m=8, nt=2048, t_window=2.0, theta=0.5, init="broadcast", fixed_iters=None),
    "c4e_m16_nt1024": twin("c4e", m=16, nt=1024, t_window=1024e-5, n_windows=1),   # CH: J̄ in the divide
}
UNFORCED = {"c6_nt8192": _c6(8192)}
CASES = {**FORCED, **UNFORCED}


@pytest.fixture
def solver_for(cuda_lib, monkeypatch):
    def make(name):
        if name in FORCED:
            monkeypatch.setenv("PARADIAG_TLONG", "1")
        return cuda_lib.Solver(CASES[name])
    return make


def _is_ch(p):
    return p.kind.startswith("cahn_hilliard")


@pytest.mark.parametrize("name", sorted(CASES))
def test_tlong_precond_parity(solver_for, name):
    p = CASES[name]
    r = np.random.default_rng(21).uniform(-1, 1, gshape(p))
    jbar = 0.137 if _is_ch(p) else 0.0
    s = solver_for(name)
    rd = to_dev(r, p)
    d = s.empty()
    s.apply_precond(rd, d, jbar)
    r_o = r.reshape(p.nt, p.nx) if p.dim == 1 else r
    d_o, _ = precond.apply_precond(p, r_o, jbar)
    # 1D: the GPU solves Step (2) in the eigenbasis (R#26).  The oracle's two exact solvers (banded
    # LU + refinement, eigenbasis divide) disagree by the instance's rounding floor f (3.4e-12 on the
    # Neumann linear-CH case, whose growing modes make d_l + μ small); the GPU is a third solver
    # with rounding of the same size, so it may sit 2f from either, on top of the generic 1e-11
    # (DESIGN.md §6).  Measured: 1.4e-11 against the LU, bar 1.7e-11.
    bar = 1e-11 + 2 * rounding_floor_1d(p, r_o, d_o) if p.dim == 1 else 1e-11
    assert rel_err(to_host(d, p), d_o) <= bar
    if p.dim == 1:
        assert rel_err(to_host(d, p), eigenbasis_precond_1d(p, r_o)) <= bar
    s.apply_precond(rd, rd, jbar)                  # in place
    assert rel_err(to_host(rd, p), d_o) <= bar


@pytest.mark.parametrize("name", sorted(CASES))
def test_tlong_solve_parity(solver_for, name):
    p = CASES[name]
    u0 = make_u0(p)
    s = solver_for(name)
    U = s.empty()
    rc, info = s.solve(to_dev(u0), U)
    U_o, iters_o, conv_o, _ = iterate.solve(p, oracle_u0(p, u0))
    assert list(info.iters[:p.n_windows]) == iters_o
    assert rel_err(to_host(U, p), U_o) <= (1e-8 if _is_ch(p) else 1e-10)
    assert info.converged == int(all(conv_o)) and rc == (0 if all(conv_o) else 1)


@pytest.mark.parametrize("nt", [1 << 15, 1 << 17])
def test_tlong_fused_pass_b_matches_unfused(cuda_lib, monkeypatch, nt):
    """N2 = 1024 splits (N_t ≥ 2^15) run pass B, the divide and pass B⁻¹ as one kernel; it must
    reproduce the three-kernel sequence (each separately pinned to the oracle above) to rounding
    (the same operations up to FMA contraction; both sit ~1e-11 from an FFT evaluation here, the
    Γ_α⁻¹ = 1/α amplification of this window's rounding floor)."""
    p = _c6(nt)
    r = np.random.default_rng(23).uniform(-1, 1, gshape(p))
    out = []
    for fuse in ("1", "0"):
        monkeypatch.setenv("PARADIAG_TLFUSE", fuse)
        s = cuda_lib.Solver(p)
        d = s.empty()
        s.apply_precond(to_dev(r, p), d, 0.0)
        out.append(to_host(d, p))
        s.close()
    assert rel_err(out[0], out[1]) <= 1e-12


def _closed_form_field(p, g, c):
    """Iterate on the whole space-time grid from its mode coefficients: u_n = T (g^{n+1} c) / 2m."""
    T = spatial.transform_matrix(p.m, p.bc)
    n = np.arange(1, p.nt + 1, dtype=np.float64)[:, None]
    G = g[None, :] ** n                              # 0 < g < 1 for θ = 1: underflows to 0, never overflows
    return (G * c[None, :]) @ T.T / (2.0 * p.m)


def test_c6_full(cuda_lib):
    """c6 at N_t = 2^20 (NEXT-3): converged iteration count and sampled iterates vs the closed-form
    per-mode WR iterate; the count is the first K whose closed-form increment meets the tolerance."""
    p = config("c6")
    u0 = make_u0(p)
    s = cuda_lib.Solver(p)
    U = s.empty()
    rc, info = s.solve(to_dev(u0), U)
    assert rc == 0
    K = int(info.iters[0])
    # closed-form stopping index: ‖U^k - U^{k-1}‖∞ ≤ tol ‖U^k‖∞
    prev = np.broadcast_to(u0.reshape(1, -1), (p.nt, p.nx))          # U⁰: u0 broadcast (R#5)
    k_cf, ratios = None, []
    for k in range(1, 10):
        cur = _closed_form_field(p, *modespace.mode_iterates(p, u0, k))
        ratio = np.abs(cur - prev).max() / np.abs(cur).max()
        ratios.append(ratio)
        if ratio <= p.tol:
            k_cf = k
            break
        prev = cur
    assert k_cf is not None and K == k_cf, (K, ratios)
    assert min(abs(np.log10(max(r, 1e-300) / p.tol)) for r in ratios) > 0.3       # no borderline stop
    Uh = to_host(U, p)
    umax = np.abs(Uh).max()
    assert abs(umax - np.abs(cur).max()) <= 1e-10 * umax
    rng = np.random.default_rng(66)
    rows = np.concatenate([rng.integers(0, p.nt, 64), [0, 1, p.nt // 2, p.nt - 1]])
    assert np.abs(Uh[rows] - cur[rows]).max() <= 1e-10 * umax
