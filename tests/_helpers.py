"""Shared test helpers: oracle-side array shapes and torch transfers (tests only)."""
import numpy as np


def gshape(p):
    return (p.nt, p.ny, p.nx)


def to_dev(a, p=None):
    import torch
    a = np.ascontiguousarray(a, dtype=np.float64)
    if p is not None:
        a = a.reshape(gshape(p))
    return torch.from_numpy(a).cuda()


def to_host(t, p=None):
    a = t.detach().cpu().numpy()
    if p is not None and p.dim == 1:
        a = a.reshape(p.nt, p.nx)
    return a


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def oracle_u0(p, u0):
    return u0.reshape(-1) if p.dim == 1 else u0


def sample_points(p, count, seed):
    rng = np.random.default_rng(seed)
    pts = [(int(rng.integers(p.nt)), int(rng.integers(p.ny)), int(rng.integers(p.nx))) for _ in range(count)]
    pts += [(p.nt - 1, 0, 0), (p.nt - 1, p.ny - 1, p.nx - 1), (0, p.ny // 2, p.nx // 2)]
    return pts


def eigenbasis_precond_1d(p, r):
    """The oracle's Step (2) solved in the eigenbasis (the method the GPU's long-window path uses)."""
    from oracle import circulant, spatial
    S1 = circulant.step1(r, p.alpha)
    d = circulant.eig_d(p.nt, p.alpha, circulant.inv_dt(p))
    e = circulant.eig_e(p.nt, p.alpha, p.theta)
    T = spatial.transform_matrix(p.m, p.bc)
    mu = spatial.mu(spatial.Lam_grid(p), p).reshape(-1)
    S2 = ((S1 @ T.T) / (d[:, None] + e[:, None] * mu[None, :])) @ T.T / (2.0 * p.m)
    d_sp, _ = circulant.step3(S2, p.alpha)
    return d_sp


def rounding_floor_1d(p, r, d_lu):
    """The rounding floor of this P_α⁻¹ instance: the oracle's own Step (2) solved a second, equally
    exact way (the eigenbasis divide the GPU uses, as oracle.precond.step2_2d does in 2D) differs
    from its banded-LU result by this much; 1D Neumann instances near the growing modes of linear
    CH (μ < 0) sit at ~3e-12."""
    return rel_err(eigenbasis_precond_1d(p, r), d_lu)
