"""GPU parity of the time-only averaged Jacobian path (NEXT-4): Step-(2) with
J̃ = diag(mean_n 3U_n²) solved by the inner GMRES of paradiag.cu (k_krylov.cuh), preconditioned
by the scalar-J̄ spectral P_α⁻¹, against the oracle's per-bin sparse direct solves
(oracle/precond.step2_2d_timeavg, pinned in tests/test_oracle_timeavg.py).
Bars: P̃⁻¹ ≤ 1e-11 relative (inner tolerance 1e-13 on the preconditioned residual); solves ≤ 1e-8
(CH, BJ) with identical per-window iteration counts."""
from dataclasses import replace

import numpy as np
import pytest

from _helpers import gshape, to_dev, to_host, rel_err
from oracle import iterate, precond
from workloads import config, twin, make_u0

pytestmark = pytest.mark.gpu

CASES = {
    "c4t_m16_nt8": twin("c4t", m=16, nt=8, t_window=8e-4, n_windows=1),
    "c4t_m32_nt16": twin("c4t", m=32, nt=16, t_window=16e-4, n_windows=2),
    "c4et_m32_nt16": replace(twin("c4e", m=32, nt=16, t_window=16e-4, n_windows=2), jacobian="time_avg"),
    "c4t_m64_nt32": twin("c4t", m=64, nt=32, t_window=32e-4, n_windows=1),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_timeavg_precond_parity(cuda_lib, name):
    p = CASES[name]
    rng = np.random.default_rng(31)
    r = rng.uniform(-1, 1, gshape(p))
    jt = 3.0 * rng.uniform(-1, 1, (p.ny, p.nx)) ** 2          # spatially varying, as mean_n 3u² is
    s = cuda_lib.Solver(p)
    d = s.empty()
    rc = s.apply_precond_jt(to_dev(r, p), d, to_dev(jt))
    assert rc == 0
    d_o, _ = precond.apply_precond(p, r, 0.0, jt)
    assert rel_err(to_host(d, p), d_o) <= 1e-11
    rd = to_dev(r, p)
    s.apply_precond_jt(rd, rd, to_dev(jt))                   # in place
    assert rel_err(to_host(rd, p), d_o) <= 1e-11


@pytest.mark.parametrize("name", sorted(CASES))
def test_timeavg_solve_parity(cuda_lib, name):
    p = CASES[name]
    u0 = make_u0(p)
    s = cuda_lib.Solver(p)
    U = s.empty()
    rc, info = s.solve(to_dev(u0), U)
    U_o, iters_o, conv_o, _ = iterate.solve(p, u0)
    assert list(info.iters[:p.n_windows]) == iters_o
    assert rel_err(to_host(U, p), U_o) <= 1e-8
    assert info.converged == int(all(conv_o))


@pytest.mark.parametrize("name", ["c4t_m32_nt16", "c4t_m64_nt32"])
def test_timeavg_device_arnoldi_matches_host_loop(cuda_lib, monkeypatch, name):
    """The inner GMRES's Arnoldi steps run as a conditional WHILE graph with the Hessenberg column,
    the Givens rotations and the stop test on the device (k_krylov.cuh, KryDev); the host loop
    (PARADIAG_KRYGRAPH=0) does the same arithmetic with the rotations on the CPU.  Both must give
    the same P̃⁻¹ r to rounding (the rotations' hypot / division may round differently)."""
    p = CASES[name]
    rng = np.random.default_rng(37)
    r = rng.uniform(-1, 1, gshape(p))
    jt = 3.0 * rng.uniform(-1, 1, (p.ny, p.nx)) ** 2
    out = []
    for g in ("1", "0"):
        monkeypatch.setenv("PARADIAG_KRYGRAPH", g)
        s = cuda_lib.Solver(p)
        d = s.empty()
        assert s.apply_precond_jt(to_dev(r, p), d, to_dev(jt)) == 0
        out.append(to_host(d, p))
        s.close()
    assert rel_err(out[0], out[1]) <= 1e-13
