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


# ---------------------------------------------------------------- pins added in round 2
@pytest.mark.parametrize("dim", [1, 2])
def test_energy_single_cosine_mode_closed_form(dim):
    """diagnostics.energy on u = A cos(kπx)(cos(lπy)) against its closed form (R#13).

    Trapezoid sums on m intervals are exact for these trigonometric polynomials:
    h Σ w cos² = 1/2, h Σ w cos⁴ = 3/8 (k, l ∉ {0, m/2, m}); each edge difference is
    -2A sin(kπ/2m) sin(kπ(2j+1)/2m), so Σ_j (δu)² = 2A² m sin²(kπ/2m).  Hence
      1D: E = ¼(3A⁴/8 - A² + 1) + ε² A² m² sin²(kπ/2m)
      2D: E = ¼(9A⁴/64 - A²/2 + 1) + (ε²/2) A² m² (sin²(kπ/2m) + sin²(lπ/2m))
    (each 2D gradient sum carries the other axis' Σ w cos² = m/2 and no h factor, h^{d-2} = 1).
    A wrong scale on the bulk or the gradient term, or a dropped weight, fails this."""
    from dataclasses import replace
    p = _ch_twin(m=32)
    if dim == 1:
        p = replace(p, dim=1)
    A, k, l = 0.7, 3, 5
    m, e2 = p.m, p.eps * p.eps
    x = np.arange(m + 1) / m
    sk, sl = np.sin(k * np.pi / (2 * m)) ** 2, np.sin(l * np.pi / (2 * m)) ** 2
    if dim == 1:
        u = A * np.cos(k * np.pi * x)
        ref = 0.25 * (3 * A ** 4 / 8 - A * A + 1) + e2 * A * A * m * m * sk
    else:
        u = A * np.outer(np.cos(l * np.pi * x), np.cos(k * np.pi * x))
        ref = 0.25 * (9 * A ** 4 / 64 - A * A / 2 + 1) + 0.5 * e2 * A * A * m * m * (sk + sl)
    assert abs(diagnostics.energy(p, u) - ref) <= 1e-14 * abs(ref)


@pytest.mark.parametrize("name,expect", [("c1", 2.03e-7), ("c2", 4.40e-2), ("c3", 1.33e-12), ("c5", 3.66)])
def test_modewise_factor_survey_probe_values(name, expect):
    """theory.modewise_factor against the survey's independent scratch probe p1."""
    f = theory.modewise_factor(config(name)).max()
    assert abs(f - expect) <= 0.005 * expect


def test_modewise_factor_is_the_per_mode_increment_ratio():
    """Per spatial mode the WR error contracts by exactly -αg^N/(1-αg^N): from the second
    iteration on both iterates are WR trajectories, so the increments δ^k_N of the physical-space
    oracle iteration, projected on the eigenmodes, have |δ^3_N / δ^2_N| = theory.modewise_factor
    mode by mode (random U⁰ excites every mode; modes whose increment is at rounding level skipped)."""
    from dataclasses import replace
    for name, kw, theta in (("c5", dict(m=16, nt=8), 1.0), ("c5", dict(m=16, nt=8), 0.5),
                            ("c2", dict(m=31, nt=8), 0.5)):
        p = replace(twin(name, theta=theta, **kw), fixed_iters=3)
        u0 = make_u0(p)
        u0 = u0.reshape(-1) if p.dim == 1 else u0
        U = np.random.default_rng(3).uniform(-1, 1, (p.nt,) + u0.shape)
        inc = []
        for _ in range(3):
            U_new, _ = iterate.iterate_once(p, u0, U)
            inc.append(U_new[-1] - U[-1])
            U = U_new
        a, b = sequential.to_modes(p, inc[1]), sequential.to_modes(p, inc[2])
        f = theory.modewise_factor(p).reshape(a.shape)
        live = np.abs(a) > 1e-6 * np.abs(a).max()
        assert live.sum() >= 20
        assert np.allclose(np.abs(b[live] / a[live]), f[live], rtol=1e-4)


@pytest.mark.parametrize("name,kw,K", [("c5", dict(m=32, nt=16), 3), ("c3", dict(m=16, nt=8), 2)])
def test_modespace_slice_values_equal_physical_iterate(name, kw, K):
    """modespace.slice_values (the whole-slice form used at full c5 size) = the physical-space
    K-th iterate of the oracle at every point of every slice."""
    from dataclasses import replace
    p = replace(twin(name, **kw), fixed_iters=K)
    u0 = make_u0(p)
    U, _, _, _ = iterate.solve(p, u0)
    g, c0 = modespace.mode_iterates(p, u0, K)
    for n in range(p.nt):
        assert np.abs(modespace.slice_values(p, g, c0, n) - U[n]).max() <= 1e-12 * np.abs(U).max()


def test_divergence_rule_stops_c5_twin():
    """BJ.c5's physics violates Thm 3.3: from U⁰ = 0 the increments grow ≈3x per
    iteration, so the SURVEY §5.3 rule stops the window unconverged after PD_GROWTH_LIMIT growths
    (iterations 1 < 2 < 3 < 4); with fixed K it only flags it.  Converging twins never trip it."""
    from dataclasses import replace
    p = replace(twin("c5", m=32, nt=16), fixed_iters=None, max_iter=50)
    hist, flags = [], []
    U, iters, conv, _ = iterate.solve(p, make_u0(p), hist, flags)
    d = [h["delta_max"] for h in hist]
    assert iters == [1 + iterate.GROWTH_LIMIT] and conv == [False] and flags == [True]
    assert all(b > a for a, b in zip(d, d[1:]))
    flags = []
    iterate.solve(replace(p, fixed_iters=6), make_u0(p), None, flags)
    assert flags == [True]
    flags = []
    q = twin("c3", m=16, nt=8)
    _, _, conv, _ = iterate.solve(q, make_u0(q), None, flags)
    assert conv == [True] and flags == [False]
