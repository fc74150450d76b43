"""Pins for oracle/iterate.py, sequential.py, modespace.py, theory.py, diagnostics.py."""
import json
import os

import numpy as np
import pytest

from oracle import iterate, sequential, modespace, theory, diagnostics, spatial
from workloads import config, twin, make_u0

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_c1_closed_form_and_count():
    """BJ.c1: sin(πx) is an eigenvector of D² (u = u_xx = 0), so BE gives u_n = (1+Δtμ₁)^{-n} sin(πx)."""
    g = json.load(open(os.path.join(GOLD, "c1_closed_form.json")))
    p = config("c1")
    m = p.m
    mu1 = 16.0 * m**4 * np.sin(np.pi / (2 * m)) ** 4
    assert abs(mu1 - g["mu1"]) <= 1e-12 * g["mu1"]
    U, iters, conv, _ = iterate.solve(p, make_u0(p))
    assert conv == [True] and iters == [g["iterations"]]
    x = np.arange(1, m) / m
    n = np.arange(1, p.nt + 1)[:, None]
    cf = (1.0 + (p.t_window / p.nt) * mu1) ** (-n) * np.sin(np.pi * x)[None, :]
    assert np.abs(U - cf).max() <= 1e-12 * np.abs(cf).max()
    assert abs(U[31, 31] - g["u_32_at_x_32_65"]) <= 1e-14
    assert abs((1.0 + (p.t_window / p.nt) * mu1) ** -32 - g["factor_n32"]) <= 1e-16


def test_c1_trapezoid_closed_form():
    """θ = ½ (NEXT-2): sin(πx) stays an eigenvector, so the converged all-at-once solution
    is u_n = R_{1/2}(Δtμ₁)^n sin(πx) with the trapezoid stability function R_{1/2}(z) =
    (1 - z/2)/(1 + z/2) — a closed form independent of the circulant machinery."""
    from dataclasses import replace
    g = json.load(open(os.path.join(GOLD, "c1_closed_form.json")))
    p = replace(config("c1"), theta=0.5)
    m = p.m
    z = (p.t_window / p.nt) * g["mu1"]
    R = (1.0 - 0.5 * z) / (1.0 + 0.5 * z)
    assert 0.0 < R < 1.0
    U, iters, conv, _ = iterate.solve(p, make_u0(p))
    assert conv == [True]
    x = np.arange(1, m) / m
    n = np.arange(1, p.nt + 1)[:, None]
    cf = R ** n * np.sin(np.pi * x)[None, :]
    assert np.abs(U - cf).max() <= 1e-12 * np.abs(cf).max()


def test_c2_fixed_point_is_sequential_solution():
    """Converged all-at-once solution = sequential BE: exact mode-wise and banded-LU stepping."""
    p = config("c2")
    u0 = make_u0(p)
    hist = []
    U, iters, conv, _ = iterate.solve(p, u0, hist)
    assert conv == [True]
    ex = sequential.exact_modewise(p, u0)
    assert np.abs(U - ex).max() <= 1e-11 * np.abs(ex).max()
    lu = sequential.lu_stepping_1d(p, u0)
    assert np.abs(lu - ex).max() <= 1e-11 * np.abs(ex).max()
    # Thm 3.3: contraction of the increments no worse than ρ (with 5% slack)
    rho = theory.thm33_rho(p)
    assert abs(rho - 0.0593) < 1e-3
    ratios = [hist[k + 1]["delta_max"] / hist[k]["delta_max"] for k in range(1, len(hist) - 2)]
    assert max(ratios) <= 1.05 * rho


@pytest.mark.parametrize("name,kw", [("c3", dict(m=32, nt=16)), ("c2", dict(m=63, nt=16)),
                                     ("c1", dict(m=17, nt=8, theta=0.5))])
def test_twin_fixed_point(name, kw):
    p = twin(name, **kw)
    u0 = make_u0(p)
    U, iters, conv, _ = iterate.solve(p, u0)
    assert conv == [True]
    ex = sequential.exact_modewise(p, u0)
    assert np.abs(U - ex).max() <= 1e-11 * np.abs(ex).max()


@pytest.mark.parametrize("theta", [1.0, 0.5])
def test_defect_correction_equals_wr_step(theta):
    """U^{k-1} + P_α⁻¹(b - K U^{k-1}) equals the direct WR solve of P:127-149 from any U^{k-1}."""
    p = twin("c2", m=6, nt=8, theta=theta, alpha=0.1)
    u0 = make_u0(p).reshape(-1)
    Uprev = np.random.default_rng(7).standard_normal((p.nt, p.nx))
    U1, _ = iterate.iterate_once(p, u0, Uprev)
    U2 = sequential.dense_wr_step(p, u0, Uprev)
    assert np.abs(U1 - U2).max() <= 1e-10 * np.abs(U2).max()


def test_residual_equals_dense_b_minus_KU():
    p = twin("c3", m=5, nt=4)
    from oracle import circulant
    u0 = make_u0(p)
    U = np.random.default_rng(8).standard_normal((p.nt, p.ny, p.nx))
    A = sequential.A_matrix(p)
    ns = A.shape[0]
    K = np.kron(circulant.C1_dense(p.nt, 0.0, circulant.inv_dt(p)), np.eye(ns)) + np.kron(np.eye(p.nt), A)
    b = np.zeros(p.nt * ns)
    b[:ns] = circulant.inv_dt(p) * u0.ravel()
    r = iterate.residual_linear(p, u0, U)
    assert np.allclose(r.ravel(), b - K @ U.ravel(), rtol=1e-12, atol=1e-9 * np.abs(b - K @ U.ravel()).max())


@pytest.mark.parametrize("name,kw,K", [("c5", dict(m=32, nt=16), 3), ("c3", dict(m=16, nt=8), 2),
                                       ("c2", dict(m=31, nt=8), 3)])
def test_modespace_closed_form_iterate(name, kw, K):
    """Closed-form per-mode WR iterate = physical-space K-th iterate."""
    p = twin(name, **kw)
    if name != "c5":
        from dataclasses import replace
        p = replace(p, fixed_iters=K)
    u0 = make_u0(p)
    U, _, _, _ = iterate.solve(p, u0)
    g, c0 = modespace.mode_iterates(p, u0, K)
    rng = np.random.default_rng(9)
    pts = [(int(rng.integers(p.nt)), int(rng.integers(p.ny)), int(rng.integers(p.nx))) for _ in range(40)]
    pts += [(p.nt - 1, 0, 0), (0, p.ny - 1, p.nx - 1)]
    ref = modespace.sample(p, g, c0, pts)
    got = np.array([U[n, iy, ix] if p.dim == 2 else U[n, ix] for n, iy, ix in pts])
    assert np.abs(ref - got).max() <= 1e-12 * np.abs(U).max()


def test_c5_theory_hypothesis_fails():
    """Thm 3.3 needs |α| R^{N_t}(z*) < 1/2; for BJ.c5 it is ≈ 2.24e10 (R#16) — fixed-K config."""
    p = config("c5")
    from oracle import circulant
    dt = 1.0 / circulant.inv_dt(p)
    b2, e2 = spatial.coeffs(p)
    zs = b2 * dt / (2 * e2)
    R = 1.0 / (1.0 + (-b2 * zs + (e2 / dt) * zs * zs))
    assert 1e10 < p.alpha * R ** p.nt < 1e11


def test_thm24_bound_biharmonic_increments():
    p = twin("c3", m=32, nt=16, alpha=0.05)
    hist = []
    iterate.solve(p, make_u0(p), hist)
    bound = theory.thm24_bound(p.alpha)
    ratios = [hist[k + 1]["delta_max"] / hist[k]["delta_max"] for k in range(1, len(hist) - 1)]
    assert ratios and max(ratios) <= 1.05 * bound


# ---------------------------------------------------------------- Cahn-Hilliard (PinT-I)
def _ch_twin(**kw):
    base = dict(m=16, nt=8, t_window=8e-4, n_windows=1)
    base.update(kw)
    return twin("c4", **base)


@pytest.mark.parametrize("c", [0.0, 1.0, -1.0])
def test_ch_constants_are_fixed_points(c):
    p = _ch_twin()
    u0 = np.full((p.ny, p.nx), c)
    U = np.full((p.nt, p.ny, p.nx), c)
    from oracle.iterate import residual_ch
    r, jbar = residual_ch(p, u0, U)
    assert np.abs(r).max() == 0.0
    assert jbar == 3 * c * c - 1


def test_ch_fixed_point_is_sequential_newton_and_dense_newton():
    from dataclasses import replace
    p = replace(_ch_twin(m=8, nt=6, t_window=6e-4), tol=1e-14, max_iter=400)
    u0 = make_u0(p)
    U, iters, conv, _ = iterate.solve(p, u0)
    seq = sequential.ch_newton_stepping(p, u0)
    assert np.abs(U - seq).max() <= 1e-11 * np.abs(seq).max()
    dense = sequential.ch_dense_newton_all_at_once(p, u0, np.broadcast_to(u0, U.shape).copy())
    assert np.abs(dense - seq).max() <= 1e-11 * np.abs(seq).max()


def test_ch_mass_and_energy():
    """Mass conservation and energy decay on the converged windows."""
    p = _ch_twin(m=32, nt=16, t_window=16e-4, n_windows=2)
    u0 = make_u0(p)
    Us = []
    u = u0
    for _ in range(p.n_windows):
        U, k, c = iterate.solve_window(p, u)
        assert c
        Us.append(U)
        u = U[-1]
    m0 = diagnostics.mass(p, u0)
    traj = [u0] + [U[n] for U in Us for n in range(p.nt)]
    masses = np.array([diagnostics.mass(p, v) for v in traj])
    assert np.abs(masses - m0).max() <= 1e-12 * max(abs(m0), 1e-3)
    E = np.array([diagnostics.energy(p, v) for v in traj])
    assert np.all(np.diff(E) <= 1e-14)
