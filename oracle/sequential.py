"""Sequential references and dense brute force (ORACLE — test infrastructure only).

* exact mode-wise θ-stepping (P:119-126 in the eigenbasis of A): U_n = T⁻¹ diag(R_θ(Δtμ)^n) T u0,
  R_θ(z) = (1 - (1-θ)z)/(1 + θz);
* banded-LU sequential stepping of (I/Δt + θA) u_n = (I/Δt - (1-θ)A) u_{n-1}, one
  nested-residual refinement per step (1D);
* dense all-at-once WR step (C1^(α)⊗I + C2^(α)⊗A) U^k = b^{k-1} (tiny sizes);
* sequential backward-Euler Newton for CH, (u_n - u_{n-1})/Δt = Δ_h(u_n³ - u_n - ε²Δ_h u_n)
   with the exact Jacobian, and the dense all-at-once Newton on G(U) (α = 0).
"""
import numpy as np
from scipy.linalg import solve_banded

from . import spatial, circulant


def _R(z, theta):
    return (1.0 - (1.0 - theta) * z) / (1.0 + theta * z)


def to_modes(prob, u: np.ndarray) -> np.ndarray:
    """Unnormalised eigen-coefficients T u (1D) or Ty u Txᵀ (2D) of the last dims."""
    T = spatial.transform_matrix(prob.m, prob.bc)
    if prob.dim == 1:
        return u @ T.T
    return T @ u @ T.T


def from_modes(prob, c: np.ndarray) -> np.ndarray:
    T = spatial.transform_matrix(prob.m, prob.bc)
    if prob.dim == 1:
        return (c @ T.T) / (2.0 * prob.m)
    return (T @ c @ T.T) / (2.0 * prob.m) ** 2


def exact_modewise(prob, u0: np.ndarray) -> np.ndarray:
    """Sequential θ-method solution u_1..u_{N_t}, exactly in the eigenbasis (linear problems)."""
    u0 = u0.reshape(-1) if prob.dim == 1 else u0
    mu = spatial.mu(spatial.Lam_grid(prob), prob)
    dt = 1.0 / circulant.inv_dt(prob)
    g = _R(dt * mu, prob.theta)
    c0 = to_modes(prob, u0)
    out = np.empty((prob.nt,) + u0.shape)
    c = c0.copy()
    for n in range(prob.nt):
        c = g * c
        out[n] = from_modes(prob, c)
    return out


def lu_stepping_1d(prob, u0: np.ndarray, refine: int = 1) -> np.ndarray:
    """Sequential θ-stepping with banded LU of the assembled I/Δt + θA (1D linear)."""
    u = u0.reshape(-1).astype(np.float64)
    n = u.size
    idt = circulant.inv_dt(prob)
    A = spatial.A_matrix_1d(prob)
    M = idt * np.eye(n) + prob.theta * A
    ab = np.zeros((5, n))
    for i in range(n):
        for j in range(max(0, i - 2), min(n, i + 3)):
            ab[2 + i - j, j] = M[i, j]
    out = np.empty((prob.nt, n))
    for k in range(prob.nt):
        rhs = idt * u - (1.0 - prob.theta) * spatial.apply_A(u, prob)
        x = solve_banded((2, 2), ab, rhs)
        for _ in range(refine):
            rho = rhs - (idt * x + prob.theta * spatial.apply_A(x, prob))
            x = x + solve_banded((2, 2), ab, rho)
        out[k] = x
        u = x
    return out


def lap_matrix(prob) -> np.ndarray:
    D = spatial.lap_matrix_1d(prob.m, prob.bc)
    if prob.dim == 1:
        return D
    I = np.eye(D.shape[0])
    return np.kron(D, I) + np.kron(I, D)        # row-major [y, x]: Δ_y ⊗ I + I ⊗ Δ_x


def A_matrix(prob) -> np.ndarray:
    L = lap_matrix(prob)
    if prob.kind == "biharmonic":
        return L @ L
    b2, e2 = spatial.coeffs(prob)
    return b2 * L + e2 * (L @ L)


def dense_wr_step(prob, u0: np.ndarray, U_prev: np.ndarray) -> np.ndarray:
    """Solve P:127-149 directly: (C1^(α)⊗I + C2^(α)⊗A) U^k = b^{k-1} (tiny sizes)."""
    nt = prob.nt
    idt = circulant.inv_dt(prob)
    A = A_matrix(prob)
    ns = A.shape[0]
    C1 = circulant.C1_dense(nt, prob.alpha, idt)
    C2 = circulant.C2_dense(nt, prob.alpha, prob.theta)
    K = np.kron(C1, np.eye(ns)) + np.kron(C2, A)
    b = np.zeros(nt * ns)
    w = u0.reshape(-1) - prob.alpha * U_prev.reshape(nt, -1)[-1]
    b[:ns] = (idt * np.eye(ns) - (1.0 - prob.theta) * A) @ w          # R#3
    return np.linalg.solve(K, b).reshape(U_prev.shape)


def dense_precond(prob, r: np.ndarray, jbar: float = 0.0) -> np.ndarray:
    """P_α⁻¹ r by a dense solve of C1^(α)⊗I + C2^(α)⊗A_eff (tiny sizes)."""
    nt = prob.nt
    idt = circulant.inv_dt(prob)
    if prob.kind == "cahn_hilliard":
        L = lap_matrix(prob)
        _, e2 = spatial.coeffs(prob)
        Aeff = -jbar * L + e2 * (L @ L)
    else:
        Aeff = A_matrix(prob)
    ns = Aeff.shape[0]
    K = np.kron(circulant.C1_dense(nt, prob.alpha, idt), np.eye(ns)) + \
        np.kron(circulant.C2_dense(nt, prob.alpha, prob.theta), Aeff)
    return np.linalg.solve(K, r.reshape(-1)).reshape(r.shape)


def dense_precond_eyre(prob, r: np.ndarray, jbar: float) -> np.ndarray:
    """PinT-II Step-(2) operator as one dense matrix (tiny sizes): C1^(α)⊗I + C3^(α)⊗Δ_h +
    I⊗(-J̄₃Δ_h + ε²Δ_h²) with C3^(α) = C2^(α) at θ = 0."""
    nt = prob.nt
    idt = circulant.inv_dt(prob)
    L = lap_matrix(prob)
    _, e2 = spatial.coeffs(prob)
    ns = L.shape[0]
    K = np.kron(circulant.C1_dense(nt, prob.alpha, idt), np.eye(ns)) + \
        np.kron(circulant.C2_dense(nt, prob.alpha, 0.0), L) + np.kron(np.eye(nt), -jbar * L + e2 * (L @ L))
    return np.linalg.solve(K, r.reshape(-1)).reshape(r.shape)


def eyre_newton_stepping(prob, u0: np.ndarray, tol: float = 1e-14, maxit: int = 50) -> np.ndarray:
    """Sequential Eyre scheme: (u_n - u_{n-1})/Δt = Δ_h u_n³ - Δ_h u_{n-1} - ε²Δ_h² u_n,
    exact-Jacobian Newton per step (tiny sizes)."""
    L = lap_matrix(prob)
    _, e2 = spatial.coeffs(prob)
    idt = circulant.inv_dt(prob)
    u = u0.reshape(-1).astype(np.float64).copy()
    ns = u.size
    out = np.empty((prob.nt, ns))
    for n in range(prob.nt):
        up = u.copy()
        x = up.copy()
        for _ in range(maxit):
            F = (x - up) * idt - L @ (x ** 3 - e2 * (L @ x)) + L @ up
            J = idt * np.eye(ns) - L @ np.diag(3.0 * x * x) + e2 * (L @ L)
            dx = np.linalg.solve(J, -F)
            x = x + dx
            if np.abs(dx).max() <= tol * max(np.abs(x).max(), 1e-300):
                break
        out[n] = x
        u = x
    return out.reshape((prob.nt,) + u0.shape)


def ch_newton_stepping(prob, u0: np.ndarray, tol: float = 1e-14, maxit: int = 50) -> np.ndarray:
    """Sequential fully implicit BE for CH, exact-Jacobian Newton per step (tiny sizes)."""
    L = lap_matrix(prob)
    _, e2 = spatial.coeffs(prob)
    idt = circulant.inv_dt(prob)
    u = u0.reshape(-1).astype(np.float64).copy()
    ns = u.size
    out = np.empty((prob.nt, ns))
    for n in range(prob.nt):
        up = u.copy()
        x = up.copy()
        for _ in range(maxit):
            F = (x - up) * idt - L @ (x ** 3 - x - e2 * (L @ x))
            J = idt * np.eye(ns) - L @ np.diag(3.0 * x * x - 1.0) + e2 * (L @ L)
            dx = np.linalg.solve(J, -F)
            x = x + dx
            if np.abs(dx).max() <= tol * max(np.abs(x).max(), 1e-300):
                break
        out[n] = x
        u = x
    return out.reshape((prob.nt,) + u0.shape)


def ch_dense_newton_all_at_once(prob, u0: np.ndarray, U_init: np.ndarray, tol=1e-14, maxit=50):
    """Full Newton on the all-at-once G(U) = 0 of P:460-463 with α = 0 (tiny sizes)."""
    L = lap_matrix(prob)
    _, e2 = spatial.coeffs(prob)
    idt = circulant.inv_dt(prob)
    nt = prob.nt
    ns = L.shape[0]
    C1 = circulant.C1_dense(nt, 0.0, idt)     # C1^(0): no corner entry
    It = np.eye(nt)
    LL = np.kron(It, L)
    X = U_init.reshape(-1).astype(np.float64).copy()
    b = np.zeros(nt * ns)
    b[:ns] = idt * u0.reshape(-1)
    Kc = np.kron(C1, np.eye(ns))
    for _ in range(maxit):
        G = Kc @ X - LL @ (X ** 3) + LL @ X + e2 * (LL @ (LL @ X)) - b
        J = Kc - LL @ np.diag(3.0 * X * X) + LL + e2 * (LL @ LL)
        dX = np.linalg.solve(J, -G)
        X = X + dX
        if np.abs(dX).max() <= tol * max(np.abs(X).max(), 1e-300):
            break
    return X.reshape(U_init.shape)
