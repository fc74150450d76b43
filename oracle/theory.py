"""Convergence factors from the paper's theorems (ORACLE — test infrastructure only).

* Thm 2.4: bound |α|/(1-|α|) for θ ∈ {1, ½}, A ⪰ 0.
* Thm 3.3: ρ = |α| R_θ^{N_t}(z*) / (1 - |α| R_θ^{N_t}(z*)),
  R_1(z) = 1/(1 + φ(z)), φ(z) = -β² z + (ε²/Δt) z², z* = β²Δt/(2ε²).
* per-mode discrete factor  W̃(z) = |α R_θ^{N_t}(z)| / |1 - α R_θ^{N_t}(z)|, z ∈ σ(ΔtA).
"""
import numpy as np

from . import spatial, circulant


def thm24_bound(alpha: float) -> float:
    return abs(alpha) / (1.0 - abs(alpha))


def thm33_rho(prob) -> float:
    dt = 1.0 / circulant.inv_dt(prob)
    b2, e2 = spatial.coeffs(prob)
    zs = b2 * dt / (2.0 * e2)
    phi = -b2 * zs + (e2 / dt) * zs * zs
    R = 1.0 / (1.0 + phi)
    q = abs(prob.alpha) * R ** prob.nt
    return q / (1.0 - q)


def modewise_factor(prob) -> np.ndarray:
    """W̃ for every spatial mode of the discrete operator (θ-method)."""
    dt = 1.0 / circulant.inv_dt(prob)
    z = dt * spatial.mu(spatial.Lam_grid(prob), prob)
    R = (1.0 - (1.0 - prob.theta) * z) / (1.0 + prob.theta * z)
    q = prob.alpha * R ** prob.nt
    return np.abs(q) / np.abs(1.0 - q)
