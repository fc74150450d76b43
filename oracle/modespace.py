"""Closed-form WR iterates per spatial mode (ORACLE — test infrastructure only).

For the linear problems the WR iteration with periodic-like initial condition (P:121-123,
eq. linear-theta1) decouples in the eigenbasis of A: for a mode with eigenvalue μ and
g = R_θ(Δtμ),
    u^k_n = g^n u^k_0,   u^k_0 = α u^k_{N_t} - α u^{k-1}_{N_t} + û0
 ⇒  u^k_0 = (û0 - α u^{k-1}_{N_t}) / (1 - α g^{N_t}).
This is the plain definition of the k-th iterate; the defect-correction form reaches the same
iterate.  Used for full-size sampled parity (c3, c5) where the physical-space
oracle would need tens of GB.
"""
import numpy as np

from . import spatial, circulant, sequential


def mode_iterates(prob, u0: np.ndarray, K: int):
    """Return (g, c0_K) with u^K_n (mode) = g^n c0_K, mode coefficients unnormalised (T u)."""
    u0 = u0.reshape(-1) if prob.dim == 1 else u0
    mu = spatial.mu(spatial.Lam_grid(prob), prob)
    dt = 1.0 / circulant.inv_dt(prob)
    g = (1.0 - (1.0 - prob.theta) * dt * mu) / (1.0 + prob.theta * dt * mu)
    c_u0 = sequential.to_modes(prob, u0)
    gN = g ** prob.nt
    if prob.init == "zero":
        last = np.zeros_like(c_u0)
    else:
        last = c_u0.copy()                  # U⁰ = u0 broadcast: u^0_{N_t} = û0
    c0 = None
    for _ in range(K):
        c0 = (c_u0 - prob.alpha * last) / (1.0 - prob.alpha * gN)
        last = gN * c0
    return g, c0


def sample(prob, g: np.ndarray, c0: np.ndarray, pts) -> np.ndarray:
    """Evaluate the iterate at sample points [(n, iy, ix)] (n = 1..N_t, 0-based array index n-1)."""
    T = spatial.transform_matrix(prob.m, prob.bc)       # T² = 2m I ⇒ T⁻¹ = T / 2m
    out = []
    for (n, iy, ix) in pts:
        c = c0 * g ** (n + 1)
        if prob.dim == 1:
            out.append(float(T[ix] @ c) / (2.0 * prob.m))
        else:
            out.append(float(T[iy] @ c @ T[ix]) / (2.0 * prob.m) ** 2)
    return np.array(out)


def slice_values(prob, g: np.ndarray, c0: np.ndarray, n: int) -> np.ndarray:
    """The whole time slice u^K_n (array index n, time level n+1) of the iterate: sample() at every
    spatial point, written as the two transform matmuls T c T / (2m)² (T symmetric)."""
    T = spatial.transform_matrix(prob.m, prob.bc)
    c = c0 * g ** (n + 1)
    if prob.dim == 1:
        return (T @ c) / (2.0 * prob.m)
    return (T @ c @ T.T) / (2.0 * prob.m) ** 2
