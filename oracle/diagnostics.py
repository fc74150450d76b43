"""Discrete mass and energy (ORACLE — test infrastructure only).

Mass ∫u and the Ginzburg-Landau energy E(u) = ∫ F(u) + (ε²/2)|∇u|², F = ¼(u²-1)²,
discretised with trapezoid weights w (½ at Neumann boundary nodes) so that wᵀΔ_h = 0 (R#13):
  mass   = h^d Σ w u
  energy = h^d Σ w F(u) + (ε²/2) h^{d-2} Σ_edges w_⊥ (u_{j+1} - u_j)²
(edge weights = the weight of the node line the edge lies on, consistent with ⟨-Δ_h u, u⟩_w).
"""
import numpy as np

from . import spatial


def _w(prob):
    w = spatial.weights_1d(prob.m, prob.bc)
    return w if prob.dim == 1 else np.outer(w, w)


def mass(prob, u: np.ndarray) -> float:
    h = 1.0 / prob.m
    return float(h ** prob.dim * np.sum(_w(prob) * u.reshape(_w(prob).shape)))


def energy(prob, u: np.ndarray) -> float:
    h = 1.0 / prob.m
    _, e2 = spatial.coeffs(prob)
    W = _w(prob)
    u = u.reshape(W.shape)
    F = 0.25 * (u * u - 1.0) ** 2
    bulk = h ** prob.dim * np.sum(W * F)
    w1 = spatial.weights_1d(prob.m, prob.bc)
    if prob.dim == 1:
        grad = np.sum(np.diff(u) ** 2) / h
    else:
        gx = np.sum(w1[:, None] * np.diff(u, axis=1) ** 2)
        gy = np.sum(w1[None, :] * np.diff(u, axis=0) ** 2)
        grad = gx + gy
    return float(bulk + 0.5 * e2 * grad)
