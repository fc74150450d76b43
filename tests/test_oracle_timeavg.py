"""Pins for the time-only averaged Jacobian oracle (NEXT-4): precond.step2_2d_timeavg /
iterate.time_avg_jacobian.  Independent of the oracle's circulant machinery: the three-step solve
equals a dense solve of the assembled all-at-once operator G̃' of P:486 (PinT-I) / its PinT-II
analogue with a random, spatially varying J̃ (so the order Δ_h·diag(J̃) is checked); a
spatially constant J̃ reduces to the scalar-J̄ path (R#8); the converged iterate is the sequential
backward-Euler (resp. Eyre) trajectory with an exact-Jacobian Newton per step."""
from dataclasses import replace

import numpy as np
import pytest

from oracle import iterate, precond, sequential, circulant, spatial
from workloads import twin, make_u0


def _ch(kind="c4", **kw):
    base = dict(m=4, nt=4, t_window=4e-4, n_windows=1, jacobian="time_avg")
    base.update(kw)
    return twin(kind, **base)


def _dense_timeavg(p, r, jt):
    """G̃' = C1^(α)⊗I + I⊗(Δ_h - Δ_h diag(jt) + ε²Δ_h²), PinT-II: C1^(α)⊗I + C3^(α)⊗Δ_h +
    I⊗(-Δ_h diag(jt) + ε²Δ_h²) with C3^(α) = C2^(α) at θ = 0; dense solve."""
    L = sequential.lap_matrix(p)
    _, e2 = spatial.coeffs(p)
    ns = L.shape[0]
    idt = circulant.inv_dt(p)
    K = np.kron(circulant.C1_dense(p.nt, p.alpha, idt), np.eye(ns))
    base = -L @ np.diag(jt.reshape(-1)) + e2 * (L @ L)
    if p.kind == "cahn_hilliard_eyre":
        K = K + np.kron(circulant.C2_dense(p.nt, p.alpha, 0.0), L) + np.kron(np.eye(p.nt), base)
    else:
        K = K + np.kron(np.eye(p.nt), L + base)
    return np.linalg.solve(K, r.reshape(-1)).reshape(r.shape)


@pytest.mark.parametrize("kind", ["c4", "c4e"])
@pytest.mark.parametrize("seed", [0, 1])
def test_three_steps_equal_dense_all_at_once(kind, seed):
    p = _ch(kind)
    rng = np.random.default_rng(seed)
    r = rng.uniform(-1, 1, (p.nt, p.ny, p.nx))
    jt = rng.uniform(0.0, 3.0, (p.ny, p.nx))            # spatially varying: Δ_h diag(jt) ≠ diag(jt) Δ_h
    d, _ = precond.apply_precond(p, r, 0.0, jt)
    ref = _dense_timeavg(p, r, jt)
    assert np.abs(d - ref).max() <= 1e-11 * np.abs(ref).max()
    # a transposed operand (diag(jt) Δ_h) is a different operator: the check above can tell
    L = sequential.lap_matrix(p)
    assert np.abs(L @ np.diag(jt.reshape(-1)) - np.diag(jt.reshape(-1)) @ L).max() > 1.0


@pytest.mark.parametrize("kind", ["c4", "c4e"])
def test_constant_jacobian_reduces_to_scalar(kind):
    p = _ch(kind, m=8, nt=8, t_window=8e-4)
    r = np.random.default_rng(3).uniform(-1, 1, (p.nt, p.ny, p.nx))
    c = 0.83
    d_t, _ = precond.apply_precond(p, r, 0.0, np.full((p.ny, p.nx), c))
    jbar = c - 1.0 if p.kind == "cahn_hilliard" else c     # J̄ = mean(3u² - 1) (R#8) / J̄₃ = mean(3u²)
    d_s, _ = precond.apply_precond(replace(p, jacobian="scalar"), r, jbar)
    assert np.abs(d_t - d_s).max() <= 1e-12 * np.abs(d_s).max()


def test_time_avg_jacobian_is_the_time_mean():
    U = np.stack([np.full((2, 2), 0.5), np.full((2, 2), -1.0), np.array([[0.0, 1.0], [2.0, 0.1]])])
    jt = iterate.time_avg_jacobian(U)
    assert np.allclose(jt, [[3 * (0.25 + 1 + 0) / 3, 3 * (0.25 + 1 + 1) / 3], [3 * (0.25 + 1 + 4) / 3, 3 * (0.25 + 1 + 0.01) / 3]],
                       rtol=0, atol=1e-15)


@pytest.mark.parametrize("kind,stepper", [("c4", sequential.ch_newton_stepping),
                                          ("c4e", sequential.eyre_newton_stepping)])
def test_converged_iterate_is_sequential_scheme(kind, stepper):
    """The fixed point does not depend on the Jacobian approximation: it is the sequential scheme."""
    p = _ch(kind, m=8, nt=8, t_window=8e-4, tol=1e-12)
    u0 = make_u0(p)
    U, iters, conv, _ = iterate.solve(p, u0)
    assert conv[0]
    ref = stepper(p, u0)
    assert np.abs(U - ref).max() <= 1e-10 * np.abs(ref).max()
