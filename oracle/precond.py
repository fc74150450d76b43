"""The preconditioner P_α⁻¹: the paper's three steps (ORACLE — test infrastructure only).

Linear problems, P:158-165 (eq. pintiter1):
  Step-(1)  S1 = (F ⊗ I)(Γ_α ⊗ I) r
  Step-(2)  S2_l = (λ_{1,l} I + λ_{2,l} A)⁻¹ S1_l,  l = 0..N_t-1   (λ_1 = d_l, λ_2 = e_l, R#1)
  Step-(3)  δ = (Γ_α⁻¹ ⊗ I)(F* ⊗ I) S2 / N_t
Cahn-Hilliard PinT-I, P:491-499 (eq. pintiter_CH): Step-(2) matrix
  λ_{1,l} I - Δ_h J̃ + Δ_h + ε²Δ_h²  with J̃ = J̄₃·I (scalar space-time mean of 3u², R#7/R#8),
  i.e. d_l I - J̄ Δ_h + ε² Δ_h² with J̄ = mean(3u² - 1).

Cahn-Hilliard PinT-II (Eyre splitting), P:537-545 (eq. pintiter_CH_eyre): Step-(2) matrix
  λ_{1,l} I - Δ_h J̃ + λ_{3,l} Δ_h + ε²Δ_h²,  λ_{3,l} = α^{1/N_t} e^{-2πil/N_t} (the eigenvalues of
  C3^(α) = C2^(α) at θ = 0), J̃ = J̄₃·I with J̄₃ = mean(3u²) (R#8); on the DCT modes the divisor is
  d_l + z ω^l Λ - J̄₃ Λ + ε² Λ².

Step-(2) solvers (a library primitive may serve as a step):
  1D: banded LU with partial pivoting (LAPACK gbsv via scipy.linalg.solve_banded) of the assembled
      pentadiagonal, then iterative refinement whose residual is evaluated in nested form (R#15)
      until the correction is below 1e-15 relative (SURVEY §8(c) oracle step 3.3).
  2D: eigenbasis of the separable Δ_h: unnormalised DST-I / DCT-I matrices (direct sums, one
      matmul per axis), divide by the mode eigenvalue, inverse transform (T² = 2m·I).
"""
import numpy as np
from scipy.linalg import solve_banded

from . import spatial, circulant


def _step2_operator_nested(prob, jbar):
    """x ↦ A_eff x in nested form, where Step-(2) solves (d_l I + e_l A_eff) x = s."""
    if prob.kind == "cahn_hilliard":
        _, e2 = spatial.coeffs(prob)

        def op(x):
            l1 = spatial.lap(x, prob.m, prob.bc, prob.dim)
            return -jbar * l1 + e2 * spatial.lap(l1, prob.m, prob.bc, prob.dim)
        return op
    return lambda x: spatial.apply_A(x, prob)


def _step2_mu(prob, jbar):
    """Eigenvalue of A_eff on the mode grid (the l-independent part for PinT-II)."""
    Lam = spatial.Lam_grid(prob)
    if prob.kind in ("cahn_hilliard", "cahn_hilliard_eyre"):
        _, e2 = spatial.coeffs(prob)
        return -jbar * Lam + e2 * (Lam * Lam)
    return spatial.mu(Lam, prob)


def _A_eff_matrix_1d(prob, jbar):
    D = spatial.lap_matrix_1d(prob.m, prob.bc)
    if prob.kind == "cahn_hilliard":
        _, e2 = spatial.coeffs(prob)
        return -jbar * D + e2 * (D @ D)
    return spatial.A_matrix_1d(prob)


def _to_banded(M: np.ndarray, kl: int, ku: int) -> np.ndarray:
    """LAPACK band storage: ab[ku + i - j, j] = M[i, j]."""
    n = M.shape[0]
    ab = np.zeros((kl + ku + 1, n), dtype=M.dtype)
    for k in range(-ku, kl + 1):                 # k = i - j
        diag = np.diagonal(M, -k)
        if k >= 0:
            ab[ku + k, :n - k] = diag
        else:
            ab[ku + k, -k:] = diag
    return ab


def step2_1d(prob, S1: np.ndarray, jbar: float = 0.0, max_refine: int = 6) -> np.ndarray:
    """Step-(2) in 1D: per bin, banded LU (partial pivoting) + nested-residual refinement."""
    nt, n = S1.shape
    d = circulant.eig_d(nt, prob.alpha, circulant.inv_dt(prob))
    e = circulant.eig_e(nt, prob.alpha, prob.theta)
    A_band = _to_banded(_A_eff_matrix_1d(prob, jbar), 2, 2)      # assembled pentadiagonal
    I_band = _to_banded(np.eye(n), 2, 2)
    op = _step2_operator_nested(prob, jbar)
    out = np.empty_like(S1)
    for l in range(nt):
        ab = d[l] * I_band + e[l] * A_band                          # d_l I + e_l A, banded
        s = S1[l]
        x = solve_banded((2, 2), ab, s)
        for _ in range(max_refine):
            Ax = op(x.real) + 1j * op(x.imag)
            rho = s - (d[l] * x + e[l] * Ax)
            c = solve_banded((2, 2), ab, rho)
            x = x + c
            if np.abs(c).max() <= 1e-15 * np.abs(x).max():
                break
        out[l] = x
    return out


def step2_2d(prob, S1: np.ndarray, jbar: float = 0.0) -> np.ndarray:
    """Step-(2) in 2D: separable eigenbasis solve per bin."""
    nt = S1.shape[0]
    d = circulant.eig_d(nt, prob.alpha, circulant.inv_dt(prob))
    e = circulant.eig_e(nt, prob.alpha, prob.theta)
    T = spatial.transform_matrix(prob.m, prob.bc)
    mu = _step2_mu(prob, jbar)                        # [q, p]
    hat = T @ S1 @ T.T                                 # Ty S Txᵀ for every bin
    denom = d[:, None, None] + e[:, None, None] * mu[None, :, :]
    if prob.kind == "cahn_hilliard_eyre":             # + λ_{3,l} Λ
        lam3 = circulant.eig_e(nt, prob.alpha, 0.0)    # e_l at θ = 0: z ω^l
        denom = denom + lam3[:, None, None] * spatial.Lam_grid(prob)[None, :, :]
    hat = hat / denom
    return (T @ hat @ T.T) / (2.0 * prob.m) ** 2


def step2_2d_timeavg(prob, S1: np.ndarray, jt: np.ndarray) -> np.ndarray:
    """Step-(2) with the paper's time-only averaged Jacobian (NEXT-4):
    J̃ = (1/N_t) Σ_n J_s(u_n) = diag(jt), jt = mean_n 3u_n² (R#7), spatially varying, so Step-(2)
    is not DCT-diagonalisable.  Per bin l the sparse system of P:495 (PinT-I)
        (λ_{1,l} I - Δ_h diag(jt) + Δ_h + ε²Δ_h²) x = S1_l
    or of P:545 (PinT-II, Eyre)
        (λ_{1,l} I - Δ_h diag(jt) + λ_{3,l} Δ_h + ε²Δ_h²) x = S1_l
    is assembled from the paper's Δ_h (Kronecker form P:284) and solved directly
    (scipy.sparse.linalg.spsolve, a library LU).  jt shaped [N_y, N_x]."""
    import scipy.sparse as sp
    from scipy.sparse.linalg import spsolve
    nt = S1.shape[0]
    d = circulant.eig_d(nt, prob.alpha, circulant.inv_dt(prob))
    _, e2 = spatial.coeffs(prob)
    D = sp.csr_matrix(spatial.lap_matrix_1d(prob.m, prob.bc))
    I1 = sp.identity(D.shape[0], format="csr")
    L = (sp.kron(D, I1) + sp.kron(I1, D)).tocsr()               # row-major [y, x]: Δ_y⊗I + I⊗Δ_x
    ns = L.shape[0]
    LJ = L @ sp.diags(jt.reshape(-1))
    base = -LJ + e2 * (L @ L)
    if prob.kind == "cahn_hilliard_eyre":
        c = circulant.eig_e(nt, prob.alpha, 0.0)                # λ_{3,l} = z ω^l
    else:
        c = np.ones(nt)                                          # + Δ_h
    I = sp.identity(ns, format="csr")
    out = np.empty(S1.shape, dtype=np.complex128)
    for l in range(nt):
        M = (d[l] * I + c[l] * L + base).tocsc()
        out[l] = spsolve(M, S1[l].reshape(-1).astype(np.complex128)).reshape(S1.shape[1:])
    return out


def apply_precond(prob, r: np.ndarray, jbar: float = 0.0, jt: np.ndarray = None):
    """δ = P_α⁻¹ r, r shaped [N_t, N_x] (1D) or [N_t, N_y, N_x] (2D).  With jt (CH, 2D): the
    time-averaged Jacobian J̃ = diag(jt) of P:486 in Step-(2) (NEXT-4) instead of the scalar J̄.

    Returns (δ, max|Im|/max|Re| after Step-(3)) — the imaginary residue of S:336.
    """
    S1 = circulant.step1(r, prob.alpha)
    if jt is not None:
        return circulant.step3(step2_2d_timeavg(prob, S1, jt), prob.alpha)
    if prob.dim == 1 and prob.kind == "cahn_hilliard_eyre":
        raise NotImplementedError("PinT-II is exercised in 2D (the library's CH path is 2D Neumann)")
    if prob.dim == 1:
        S2 = step2_1d(prob, S1, jbar)
    else:
        S2 = step2_2d(prob, S1, jbar)
    return circulant.step3(S2, prob.alpha)
