"""Pins for oracle/precond.py: the three steps vs a dense all-at-once solve."""
import numpy as np
import pytest

from oracle import precond, sequential
from workloads import twin

CASES = [
    ("c1", dict(m=7, nt=4)),
    ("c1", dict(m=9, nt=8, theta=0.5)),
    ("c2", dict(m=7, nt=8)),
    ("c2", dict(m=6, nt=4, theta=0.5, alpha=0.2)),
    ("c3", dict(m=6, nt=8)),
    ("c3", dict(m=5, nt=4, theta=0.5)),
    ("c5", dict(m=4, nt=4)),
    ("c5", dict(m=5, nt=8, alpha=0.3)),
]


@pytest.mark.parametrize("name,kw", CASES)
def test_three_steps_equal_dense_solve(name, kw):
    p = twin(name, **kw)
    shape = (p.nt, p.nx) if p.dim == 1 else (p.nt, p.ny, p.nx)
    r = np.random.default_rng(4).standard_normal(shape)
    d1, imag = precond.apply_precond(p, r)
    d2 = sequential.dense_precond(p, r)
    assert np.abs(d1 - d2).max() <= 1e-10 * np.abs(d2).max()
    assert imag < 1e-11


@pytest.mark.parametrize("jbar", [-1.0, -0.3, 0.0, 0.8, 2.0])
def test_ch_step2_equals_dense(jbar):
    # P:495 Step-(2) matrix λ_1 I - Δ_h J̃ + Δ_h + ε²Δ_h² with scalar J̃ (R#8).
    p = twin("c4", m=5, nt=4, alpha=0.05)
    r = np.random.default_rng(5).standard_normal((p.nt, p.ny, p.nx))
    d1, _ = precond.apply_precond(p, r, jbar)
    d2 = sequential.dense_precond(p, r, jbar)
    assert np.abs(d1 - d2).max() <= 1e-10 * np.abs(d2).max()


def test_1d_refinement_reaches_spectral_accuracy():
    # c2's bin 0 has cond ≈ 1e10; LU + nested refinement must agree with the eigenbasis solve.
    p = twin("c2", m=1023, nt=4)
    r = np.random.default_rng(6).standard_normal((p.nt, p.nx))
    from oracle import circulant, spatial
    S1 = circulant.step1(r, p.alpha)
    x1 = precond.step2_1d(p, S1)
    T = spatial.transform_matrix(p.m, p.bc)
    d = circulant.eig_d(p.nt, p.alpha, circulant.inv_dt(p))
    mu = spatial.mu(spatial.lambdas(p.m, p.bc), p)
    x2 = ((S1 @ T.T) / (d[:, None] + mu[None, :])) @ T.T / (2 * p.m)
    assert np.abs(x1 - x2).max() <= 1e-10 * np.abs(x2).max()
