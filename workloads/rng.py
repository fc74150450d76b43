"""splitmix64 counter-based generator and the u0 recipes (SURVEY.md §8(d) RNG contract).

Contract (both sides):
  state_i = seed + (i+1) * 0x9E3779B97F4A7C15  (mod 2^64), i = 0, 1, ...
  z = state_i; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
               z = (z ^ (z >> 27)) * 0x94D049BB133111EB
               z =  z ^ (z >> 31)
  u = (z >> 11) * 2^-53 in [0, 1);   value = a + (b - a) * u
  fill order: row-major over the unknowns (y outer, x inner).
"""
import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, n: int) -> np.ndarray:
    """First n outputs of splitmix64 seeded with `seed` (uint64 array)."""
    with np.errstate(over="ignore"):
        i = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed: int, n: int, a: float, b: float) -> np.ndarray:
    u = (splitmix64(seed, n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return a + (b - a) * u


def grid_coords(m: int, bc: str) -> np.ndarray:
    """Node coordinates along one axis of (0,1) with h = 1/m.

    Neumann: nodes j = 0..m (m+1 unknowns, boundary nodes included).
    Hinged (u = Δu = 0, P:703 case (ii)): interior j = 1..m-1.
    """
    if bc == "neumann":
        j = np.arange(0, m + 1)
    elif bc == "hinged":
        j = np.arange(1, m)
    else:
        raise ValueError(bc)
    return j / m


def make_u0(prob) -> np.ndarray:
    """Initial data u0 for a Problem, shape [ny][nx] (ny = 1 in 1D), float64."""
    x = grid_coords(prob.m, prob.bc)
    n = x.size
    shape = (n, n) if prob.dim == 2 else (1, n)
    kind = prob.u0_kind
    if kind == "sine":
        if prob.dim == 1:
            return np.sin(np.pi * x)[None, :].copy()
        return np.sin(np.pi * x)[:, None] * np.sin(np.pi * x)[None, :]
    if kind == "uniform":
        a, b = prob.u0_range
        return uniform(prob.seed, shape[0] * shape[1], a, b).reshape(shape)
    if kind == "sine_plus_noise":
        a, b = prob.u0_range
        base = np.sin(np.pi * x)[:, None] * np.sin(np.pi * x)[None, :] if prob.dim == 2 \
            else np.sin(np.pi * x)[None, :]
        return base + uniform(prob.seed, shape[0] * shape[1], a, b).reshape(shape)
    if kind == "constant":
        return np.full(shape, prob.u0_range[0])
    raise ValueError(kind)
