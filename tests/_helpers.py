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
