"""Pins for oracle/spatial.py against the paper's printed matrix and library eigensolvers."""
import numpy as np
import pytest

from oracle import spatial
from workloads import twin


def test_neumann_matrix_is_paper_deltah():
    # Δ_h = (1/h²) [[-2, 2], [1, -2, 1], ..., [2, -2]]
    m = 5
    D = spatial.lap_matrix_1d(m, "neumann") / m**2
    expect = np.array([[-2, 2, 0, 0, 0, 0],
                       [1, -2, 1, 0, 0, 0],
                       [0, 1, -2, 1, 0, 0],
                       [0, 0, 1, -2, 1, 0],
                       [0, 0, 0, 1, -2, 1],
                       [0, 0, 0, 0, 2, -2]], float)
    assert np.array_equal(D, expect)


@pytest.mark.parametrize("bc", ["neumann", "hinged"])
def test_nested_equals_matrix_1d(bc):
    m = 9
    D = spatial.lap_matrix_1d(m, bc)
    u = np.random.default_rng(0).standard_normal(spatial.n_unknowns(m, bc))
    assert np.allclose(spatial.lap(u, m, bc, 1), D @ u, rtol=1e-13, atol=1e-10)


@pytest.mark.parametrize("bc", ["neumann", "hinged"])
def test_nested_equals_kron_2d(bc):
    m = 6
    D = spatial.lap_matrix_1d(m, bc)
    n = D.shape[0]
    L = np.kron(D, np.eye(n)) + np.kron(np.eye(n), D)      # I⊗Δ_h + Δ_h⊗I
    u = np.random.default_rng(1).standard_normal((n, n))
    assert np.allclose(spatial.lap(u, m, bc, 2).ravel(), L @ u.ravel(), rtol=1e-13, atol=1e-10)


def test_neumann_invariants_exact():
    # Δ_h·1 = 0 and wᵀΔ_h = 0 exactly: mass conservation of the discrete operator.
    for m in (4, 7, 64):
        D = spatial.lap_matrix_1d(m, "neumann")
        w = spatial.weights_1d(m, "neumann")
        assert np.all(D @ np.ones(m + 1) == 0.0)
        assert np.all(w @ D == 0.0)


def test_hinged_biharmonic_rows():
    # u = Δu = 0 (P:703 (ii)) ⇒ A = D² with rows ×h⁴ (5,-4,1), (-4,6,-4,1), (1,-4,6,-4,1)
    m = 8
    D = spatial.lap_matrix_1d(m, "hinged") / m**2
    A = D @ D
    assert np.array_equal(A[0, :3], [5, -4, 1])
    assert np.array_equal(A[1, :4], [-4, 6, -4, 1])
    assert np.array_equal(A[3, 1:6], [1, -4, 6, -4, 1])


@pytest.mark.parametrize("bc", ["neumann", "hinged"])
@pytest.mark.parametrize("m", [4, 7, 11])
def test_spectrum_vs_library_eigensolver(bc, m):
    D = spatial.lap_matrix_1d(m, bc)
    ev = np.sort(np.linalg.eigvals(D).real)
    lam = np.sort(spatial.lambdas(m, bc))
    assert np.allclose(ev, lam, rtol=1e-10, atol=1e-9 * m * m)


def test_spectrum_matches_paper_cos_form():
    # λ_p = (2/h²){cos((p-1)π/(N_x-1)) - 1}, p = 1..N_x, N_x = m+1 nodes
    m = 16
    p = np.arange(1, m + 2)
    paper = 2.0 * m * m * (np.cos((p - 1) * np.pi / m) - 1.0)
    assert np.allclose(spatial.lambdas(m, "neumann"), paper, rtol=1e-12, atol=1e-10)


@pytest.mark.parametrize("bc", ["neumann", "hinged"])
def test_transform_diagonalises(bc):
    m = 8
    T = spatial.transform_matrix(m, bc)
    D = spatial.lap_matrix_1d(m, bc)
    assert np.allclose(T @ T, 2 * m * np.eye(T.shape[0]), atol=1e-12)
    assert np.allclose(T @ D @ T / (2 * m), np.diag(spatial.lambdas(m, bc)), atol=1e-9)


def test_linear_ch_operator():
    p = twin("c2", m=8)
    D = spatial.lap_matrix_1d(8, "neumann")
    u = np.random.default_rng(2).standard_normal(9)
    A = p.beta**2 * D + p.eps**2 * D @ D
    assert np.allclose(spatial.apply_A(u, p), A @ u, rtol=1e-12, atol=1e-9)
