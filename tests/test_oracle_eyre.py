"""Pins for the PinT-II (Eyre convex splitting) oracle, NEXT-1: oracle/iterate.py
residual_ch_eyre, precond (Step-(2) with λ_{3,l}Δ_h), sequential.eyre_newton_stepping /
dense_precond_eyre.  Pins independent of the oracle's circulant machinery: constant states are
exact fixed points, the three-step solve equals a dense solve of the assembled P:533-536 operator,
the converged all-at-once iterate equals sequential Eyre stepping with an exact-Jacobian Newton per
step, and the Eyre trajectory conserves mass and does not increase the discrete energy."""
from dataclasses import replace

import numpy as np
import pytest

from oracle import iterate, precond, sequential, diagnostics
from oracle.iterate import residual_ch_eyre
from workloads import twin, make_u0


def _eyre(**kw):
    base = dict(m=16, nt=8, t_window=8e-4, n_windows=1)
    base.update(kw)
    return twin("c4e", **base)


@pytest.mark.parametrize("c", [0.0, 1.0, -1.0, 0.37])
def test_constants_are_fixed_points(c):
    # Δ_h annihilates constants, so r ≡ 0 exactly; J̄₃ = 3c²
    p = _eyre()
    u0 = np.full((p.ny, p.nx), c)
    U = np.full((p.nt, p.ny, p.nx), c)
    r, jbar = residual_ch_eyre(p, u0, U)
    assert np.abs(r).max() == 0.0
    assert abs(jbar - 3 * c * c) <= 1e-15


def test_residual_matches_sequential_scheme():
    # r_n = -( (U_n - U_{n-1})/Δt - Δ_h U_n³ + Δ_h U_{n-1} + ε²Δ_h² U_n ) assembled with dense Δ_h
    p = _eyre(m=6, nt=3)
    rng = np.random.default_rng(3)
    u0 = rng.uniform(-1, 1, (p.ny, p.nx))
    U = rng.uniform(-1, 1, (p.nt, p.ny, p.nx))
    r, jbar = residual_ch_eyre(p, u0, U)
    L = sequential.lap_matrix(p)
    e2 = p.eps * p.eps
    idt = p.nt / p.t_window
    prev = u0.reshape(-1)
    for n in range(p.nt):
        x = U[n].reshape(-1)
        ref = -((x - prev) * idt - L @ x ** 3 + L @ prev + e2 * (L @ (L @ x)))
        assert np.abs(r[n].reshape(-1) - ref).max() <= 1e-11 * np.abs(ref).max()
        prev = x
    assert abs(jbar - 3.0 * np.mean(U * U)) <= 1e-15


@pytest.mark.parametrize("jbar", [0.0, 0.5, 1.7, 3.0])
def test_step2_equals_dense(jbar):
    # Step-(2) matrix λ_1 I - Δ_h J̃ + λ_3 Δ_h + ε²Δ_h² with scalar J̃ (R#8)
    p = twin("c4e", m=5, nt=4, alpha=0.05)
    r = np.random.default_rng(5).standard_normal((p.nt, p.ny, p.nx))
    d1, imag = precond.apply_precond(p, r, jbar)
    d2 = sequential.dense_precond_eyre(p, r, jbar)
    assert np.abs(d1 - d2).max() <= 1e-10 * np.abs(d2).max()
    assert imag < 1e-11


def test_fixed_point_is_sequential_eyre():
    p = replace(_eyre(m=8, nt=6, t_window=6e-4), tol=1e-14, max_iter=400)
    u0 = make_u0(p)
    U, iters, conv, _ = iterate.solve(p, u0)
    assert conv == [True]
    seq = sequential.eyre_newton_stepping(p, u0)
    assert np.abs(U - seq).max() <= 1e-11 * np.abs(seq).max()
    # the Eyre trajectory differs from the fully implicit one (a different scheme)
    be = sequential.ch_newton_stepping(replace(p, kind="cahn_hilliard"), u0)
    assert np.abs(be - seq).max() > 1e-8 * np.abs(seq).max()


def test_mass_and_energy():
    """Eyre's scheme is unconditionally energy stable: along the converged windows the
    weighted mass is constant and the discrete energy does not increase."""
    p = _eyre(m=32, nt=16, t_window=16e-4, n_windows=2)
    u0 = make_u0(p)
    traj, u = [u0], u0
    for _ in range(p.n_windows):
        U, k, c = iterate.solve_window(p, u)
        assert c
        traj += [U[n] for n in range(p.nt)]
        u = U[-1]
    m0 = diagnostics.mass(p, u0)
    masses = np.array([diagnostics.mass(p, v) for v in traj])
    assert np.abs(masses - m0).max() <= 1e-12 * max(abs(m0), 1e-3)
    E = np.array([diagnostics.energy(p, v) for v in traj])
    assert np.all(np.diff(E) <= 1e-14)
