"""Spatial finite-difference operators (ORACLE — test infrastructure only).

* Neumann Δ_h (paper eq. deltah): vertex grid j = 0..m, h = 1/m,
  ghost reflection u_{-1} = u_1, u_{m+1} = u_{m-1}; matrix rows (-2, 2), (1,-2,1), (2,-2) / h².
* Hinged, u = Δu = 0 (P:701-705 case (ii), R#14): interior j = 1..m-1, zero ghosts at each
  Laplacian application, so A = D² (1D) and (D⊗I + I⊗D)² (2D).
* 2D Laplacian I⊗Δ_h + Δ_h⊗I.
* A = Δ_h² (biharmonic), A = β²Δ_h + ε²Δ_h² (linearised CH).

Nested evaluation (R#15): L(u) = ((u_W + u_E) + (u_S + u_N) - 4 u_C) * m², and
A u = L(L(u)) or β²·L(u) + ε²·L(L(u)); 1/h² = m² exactly, β² = fl(β·β), ε² = fl(ε·ε) (R#20).
"""
import numpy as np


def n_unknowns(m: int, bc: str) -> int:
    return m + 1 if bc == "neumann" else m - 1


def _pad(u: np.ndarray, axis: int, bc: str) -> np.ndarray:
    """Append one ghost layer on each side of `axis` (P:110-117 reflection or zero)."""
    u = np.moveaxis(u, axis, -1)
    if bc == "neumann":
        lo, hi = u[..., 1:2], u[..., -2:-1]          # u_{-1} = u_1, u_{m+1} = u_{m-1}
    elif bc == "hinged":
        lo, hi = np.zeros_like(u[..., :1]), np.zeros_like(u[..., :1])   # u_0 = u_m = 0
    else:
        raise ValueError(bc)
    return np.moveaxis(np.concatenate([lo, u, hi], axis=-1), -1, axis)


def lap(u: np.ndarray, m: int, bc: str, dim: int) -> np.ndarray:
    """Nested discrete Laplacian of the last `dim` axes of u (R#15)."""
    inv_h2 = float(m) * float(m)
    if dim == 1:
        p = _pad(u, -1, bc)
        return ((p[..., :-2] + p[..., 2:]) - 2.0 * u) * inv_h2
    px = _pad(u, -1, bc)
    py = _pad(u, -2, bc)
    we = px[..., :-2] + px[..., 2:]
    sn = py[..., :-2, :] + py[..., 2:, :]
    return ((we + sn) - 4.0 * u) * inv_h2


def coeffs(prob):
    """(β², ε²) rounded once from the double inputs (R#20)."""
    return prob.beta * prob.beta, prob.eps * prob.eps


def apply_A(u: np.ndarray, prob) -> np.ndarray:
    """A u in nested form: biharmonic A = Δ_h²; linearised CH A = β²Δ_h + ε²Δ_h²."""
    l1 = lap(u, prob.m, prob.bc, prob.dim)
    l2 = lap(l1, prob.m, prob.bc, prob.dim)
    if prob.kind == "biharmonic":
        return l2
    if prob.kind == "linear_ch":
        b2, e2 = coeffs(prob)
        return b2 * l1 + e2 * l2
    raise ValueError("apply_A is for the linear problems; CH uses iterate.residual_ch")


def lap_matrix_1d(m: int, bc: str) -> np.ndarray:
    """Dense 1D Laplacian matrix: Neumann = the paper's Δ_h printed at P:109-118."""
    n = n_unknowns(m, bc)
    D = np.zeros((n, n))
    for i in range(n):
        D[i, i] = -2.0
        if i > 0:
            D[i, i - 1] = 1.0
        if i < n - 1:
            D[i, i + 1] = 1.0
    if bc == "neumann":
        D[0, 1] = 2.0          # first row (-2, 2)
        D[n - 1, n - 2] = 2.0  # last row (2, -2)
    return D * (float(m) * float(m))


def A_matrix_1d(prob) -> np.ndarray:
    """Dense 1D A (assembled; for LU factorisation and tiny dense pins only)."""
    D = lap_matrix_1d(prob.m, prob.bc)
    if prob.kind == "biharmonic":
        return D @ D
    b2, e2 = coeffs(prob)
    return b2 * D + e2 * (D @ D)


def lambdas(m: int, bc: str) -> np.ndarray:
    """Eigenvalues of the 1D Δ_h, λ_p = -4 m² sin²(pπ/(2m)) (R#11; = P:233 for Neumann).

    Neumann: p = 0..m (eigenvector cos(pπj/m)); hinged: p = 1..m-1 (eigenvector sin(pπj/m)).
    """
    p = np.arange(0, m + 1) if bc == "neumann" else np.arange(1, m)
    s = np.sin(p * np.pi / (2.0 * m))
    return -4.0 * (float(m) * float(m)) * s * s


def mu(Lam: np.ndarray, prob) -> np.ndarray:
    """Eigenvalue of A for a Laplacian eigenvalue Λ."""
    if prob.kind == "biharmonic":
        return Lam * Lam
    b2, e2 = coeffs(prob)
    return b2 * Lam + e2 * (Lam * Lam)


def Lam_grid(prob) -> np.ndarray:
    """Laplacian eigenvalues on the mode grid: 1D λ_p, 2D λ_{p,q} = λ_p + λ_q."""
    lam = lambdas(prob.m, prob.bc)
    if prob.dim == 1:
        return lam
    return lam[:, None] + lam[None, :]      # [q (y), p (x)]


def transform_matrix(m: int, bc: str) -> np.ndarray:
    """Unnormalised eigenbasis transform T of the 1D Δ_h, with T @ T = 2m·I.

    Neumann: DCT-I, T[p, j] = c_j cos(π p j / m), c_j = 1 for j in {0, m} else 2 (REDFT00).
    Hinged:  DST-I, T[p, j] = 2 sin(π p j / m), p, j = 1..m-1 (RODFT00).
    The angle uses the exact integer reduction (p·j) mod 2m.
    """
    if bc == "neumann":
        idx = np.arange(0, m + 1)
        k = np.outer(idx, idx) % (2 * m)
        T = np.cos(np.pi * k / m)
        T[:, 1:m] *= 2.0
        return T
    idx = np.arange(1, m)
    k = np.outer(idx, idx) % (2 * m)
    return 2.0 * np.sin(np.pi * k / m)


def weights_1d(m: int, bc: str) -> np.ndarray:
    """Trapezoid weights w (½ at Neumann boundary nodes) with wᵀΔ_h = 0 (R#13)."""
    n = n_unknowns(m, bc)
    w = np.ones(n)
    if bc == "neumann":
        w[0] = w[-1] = 0.5
    return w
