"""Pins for oracle/circulant.py: Lemma 2.1 reconstruction and the Step-(1)/(3) round trip."""
import numpy as np
import pytest

from oracle import circulant


@pytest.mark.parametrize("nt", [2, 5, 8, 16, 64])
@pytest.mark.parametrize("alpha", [1e-3, 0.05, 0.5])
@pytest.mark.parametrize("theta", [1.0, 0.5])
def test_lemma21_reconstruction(nt, alpha, theta):
    # C_j = V D_j V^{-1}, V = Γ_α⁻¹ F* (our F has the e^{-2πi} sign, R#1).
    idt = 7.0
    g = circulant.gamma(nt, alpha)
    F = circulant.dft_matrix(nt)
    V = np.diag(1.0 / g) @ np.conj(F) / nt
    Vinv = F @ np.diag(g)
    assert np.allclose(V @ Vinv, np.eye(nt), atol=1e-12)
    C1 = circulant.C1_dense(nt, alpha, idt)
    C2 = circulant.C2_dense(nt, alpha, theta)
    d = circulant.eig_d(nt, alpha, idt)
    e = circulant.eig_e(nt, alpha, theta)
    for C, lam in ((C1, d), (C2, e)):
        R = V @ np.diag(lam) @ Vinv
        assert np.linalg.norm(R - C) <= 1e-10 * np.linalg.norm(C)


def test_eigenvalues_from_first_column():
    # D_j = diag(√N_t F Γ_α C_j(:,1)) with the paper's unitary F — same values, our sign.
    nt, alpha, idt = 8, 0.01, 3.0
    C1 = circulant.C1_dense(nt, alpha, idt)
    col = C1[:, 0]
    g = circulant.gamma(nt, alpha)
    D = circulant.dft_matrix(nt) @ (g * col)
    assert np.allclose(D, circulant.eig_d(nt, alpha, idt), atol=1e-13)


def test_pairing_identity():
    # d_l Δt + z ω^l = 1
    nt, alpha, idt = 32, 1e-4, 320.0
    z = alpha ** (1.0 / nt)
    d = circulant.eig_d(nt, alpha, idt)
    assert np.allclose(d / idt + z * circulant.omega_pow(nt), 1.0, atol=1e-15)


def test_step3_inverts_step1():
    r = np.random.default_rng(3).standard_normal((16, 5, 3))
    back, imag = circulant.step3(circulant.step1(r, 1e-3), 1e-3)
    assert np.allclose(back, r, atol=1e-12) and imag < 1e-12


def test_gamma_indexing():
    # Γ_α = diag(1, α^{1/N_t}, …, α^{(N_t-1)/N_t}): first entry exactly 1
    g = circulant.gamma(4, 1e-4)
    assert g[0] == 1.0 and np.isclose(g[2], 1e-4 ** 0.5, rtol=1e-14)
