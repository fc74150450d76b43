"""α-circulant time matrices and their diagonalisation (ORACLE — test infrastructure only).

C1^(α), C2^(α): P:131-146 (eq. ciculantmat).  Lemma 2.1: C_j = V D_j V⁻¹ with
V = Γ_α⁻¹ F*, Γ_α = diag(α^{(l-1)/N_t}).

Readings:
  R#1  forward DFT kernel e^{-2πi jl/N_t} (FFTW sign), so the eigenvalues that go with it are
       d_l = (1 - z ω^l)/Δt,  e_l = θ + (1-θ) z ω^l,  z = α^{1/N_t}, ω = e^{-2πi/N_t}
       (P:166-168 with the 1/Δt of C1 kept).
  R#2  γ_j = α^{j/N_t} for 0-based j = n-1, computed as exp(j·ln α / N_t).
  R#20 1/Δt := N_t / T.
"""
import numpy as np


def inv_dt(prob) -> float:
    return prob.nt / prob.t_window


def gamma(nt: int, alpha: float) -> np.ndarray:
    """γ_j = α^{j/N_t}, j = 0..N_t-1 (Γ_α of P:156, R#2)."""
    j = np.arange(nt)
    return np.exp(j * np.log(alpha) / nt)


def omega_pow(nt: int) -> np.ndarray:
    """ω^l = e^{-2πi l/N_t}, l = 0..N_t-1."""
    l = np.arange(nt)
    return np.exp(-2j * np.pi * l / nt)


def eig_d(nt: int, alpha: float, inv_dt_: float) -> np.ndarray:
    """Eigenvalues of C1^(α): d_l = (1 - z ω^l)/Δt (P:168 λ_{1,n} with 1/Δt, R#1)."""
    z = np.exp(np.log(alpha) / nt)
    return (1.0 - z * omega_pow(nt)) * inv_dt_


def eig_e(nt: int, alpha: float, theta: float) -> np.ndarray:
    """Eigenvalues of C2^(α): e_l = θ + (1-θ) z ω^l (P:168 λ_{2,n})."""
    z = np.exp(np.log(alpha) / nt)
    return theta + (1.0 - theta) * z * omega_pow(nt)


def dft_matrix(nt: int) -> np.ndarray:
    """Unnormalised forward DFT F[l, j] = exp(-2πi ((l·j) mod N_t)/N_t) (exact index reduction)."""
    idx = np.arange(nt)
    k = np.outer(idx, idx) % nt
    return np.exp(-2j * np.pi * k / nt)


def C1_dense(nt: int, alpha: float, inv_dt_: float) -> np.ndarray:
    """C1^(α) of P:132-138."""
    C = np.eye(nt)
    for j in range(1, nt):
        C[j, j - 1] = -1.0
    C[0, nt - 1] = -alpha
    return C * inv_dt_


def C2_dense(nt: int, alpha: float, theta: float) -> np.ndarray:
    """C2^(α) of P:139-145."""
    C = theta * np.eye(nt)
    for j in range(1, nt):
        C[j, j - 1] = 1.0 - theta
    C[0, nt - 1] = (1.0 - theta) * alpha
    return C


def step1(r: np.ndarray, alpha: float) -> np.ndarray:
    """Step-(1) of P:161: S1 = (F ⊗ I)(Γ_α ⊗ I) r, time on axis 0 (naive O(N_t²) DFT by matmul)."""
    nt = r.shape[0]
    g = gamma(nt, alpha).reshape((nt,) + (1,) * (r.ndim - 1))
    s = (g * r).reshape(nt, -1)
    return (dft_matrix(nt) @ s).reshape(r.shape)


def step3(x: np.ndarray, alpha: float):
    """Step-(3) of P:163: U = (Γ_α⁻¹ ⊗ I)(F* ⊗ I) S2 / N_t.  Returns (real part, max|imag|/max|real|)."""
    nt = x.shape[0]
    F = dft_matrix(nt)
    y = (np.conj(F) @ x.reshape(nt, -1)).reshape(x.shape) / nt
    g = gamma(nt, alpha).reshape((nt,) + (1,) * (x.ndim - 1))
    y = y / g
    scale = max(np.abs(y.real).max(), 1e-300)
    return y.real.copy(), float(np.abs(y.imag).max() / scale)
