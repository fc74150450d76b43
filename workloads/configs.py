"""Problem parameter tables: BASELINE.json configs c1..c5 plus reduced twins.

Readings: 1D sizes as stated; 2D "N×N grid" = N intervals (h = 1/N),
so Neumann has N+1 nodes per axis and hinged has N-1 interior unknowns per axis.
Δt = T/Nt.  U⁰ = u0 broadcast (c1-c4) or 0 (c5, fixed K = 3 iterations).
"""
from dataclasses import dataclass, replace, field
from typing import Optional, Tuple


@dataclass(frozen=True)
class Problem:
    name: str
    kind: str            # "biharmonic" | "linear_ch" | "cahn_hilliard" (PinT-I) | "cahn_hilliard_eyre" (PinT-II)
    bc: str              # "neumann" | "hinged"
    dim: int             # 1 or 2
    m: int               # intervals per axis, h = 1/m
    nt: int              # time steps per window
    t_window: float      # window length T (Δt = t_window / nt)
    alpha: float
    theta: float = 1.0
    beta: float = 0.0
    eps: float = 0.0
    n_windows: int = 1
    tol: float = 1e-10
    max_iter: int = 100
    omega: float = 1.0   # damping cap: ω_k = min(omega, tau / ||δ||∞)
    tau: float = float("inf")
    init: str = "broadcast"          # "broadcast" | "zero"
    fixed_iters: Optional[int] = None  # run exactly K iterations (c5)
    u0_kind: str = "uniform"
    u0_range: Tuple[float, float] = (0.0, 0.0)
    seed: int = 0
    jacobian: str = "scalar"         # CH: "scalar" J̄ (R#8) | "time_avg" J̃ = diag(mean_n 3u_n²) (NEXT-4)

    @property
    def n(self) -> int:
        """Unknowns per axis."""
        return self.m + 1 if self.bc == "neumann" else self.m - 1

    @property
    def nx(self) -> int:
        return self.n

    @property
    def ny(self) -> int:
        return self.n if self.dim == 2 else 1

    @property
    def ns(self) -> int:
        return self.nx * self.ny

    @property
    def dofs(self) -> int:
        return self.nt * self.ns


CONFIGS = {
    # BJ.c1: 1D biharmonic, u = u_xx = 0, 64 interior points (h = 1/65), Nt = 32, T = 0.1
    "c1": Problem("c1", "biharmonic", "hinged", 1, m=65, nt=32, t_window=0.1, alpha=1e-3,
                  tol=1e-12, u0_kind="sine"),
    # BJ.c2: 1D linearised CH, Neumann, 1024 nodes (h = 1/1023), Nt = 256, T = 1
    "c2": Problem("c2", "linear_ch", "neumann", 1, m=1023, nt=256, t_window=1.0, alpha=1e-4,
                  beta=0.5, eps=0.05, u0_range=(-0.05, 0.05), seed=2),
    # BJ.c3: 2D biharmonic, u = Δu = 0, 512x512 grid -> 511^2 interior, Nt = 128, T = 0.05
    "c3": Problem("c3", "biharmonic", "hinged", 2, m=512, nt=128, t_window=0.05, alpha=1e-4,
                  u0_kind="sine_plus_noise", u0_range=(-0.01, 0.01), seed=3),
    # BJ.c4: 2D CH PinT-I, Neumann, 256x256 grid -> 257^2 nodes, Nt = 64 per window, Δt = 1e-4
    "c4": Problem("c4", "cahn_hilliard", "neumann", 2, m=256, nt=64, t_window=64e-4, alpha=1e-3,
                  eps=0.02, n_windows=4, max_iter=400, omega=0.7, tau=1.0,
                  u0_range=(-0.1, 0.1), seed=4),
    # BJ.c5: 2D linearised CH, Neumann, 2048x2048 grid -> 2049^2 nodes, Nt = 512, T = 0.5
    "c5": Problem("c5", "linear_ch", "neumann", 2, m=2048, nt=512, t_window=0.5, alpha=1e-4,
                  beta=0.4, eps=0.01, init="zero", fixed_iters=3,
                  u0_range=(-0.05, 0.05), seed=5),
    # NEXT-1: c4's physics and windows solved with PinT-II (Eyre convex splitting,
    # P:502-545) — the scheme the paper runs for its 2D CH experiments
    "c4e": Problem("c4e", "cahn_hilliard_eyre", "neumann", 2, m=256, nt=64, t_window=64e-4, alpha=1e-3,
                   eps=0.02, n_windows=4, max_iter=400, omega=0.7, tau=1.0,
                   u0_range=(-0.1, 0.1), seed=4),
    # NEXT-3: the long-window 1D run "Δt = 10⁻⁶, i.e. N_t = 10⁶ ... four
    # iterations", h = 1/64, T = 1, α = 10⁻³ (Fig. 3).  Power-of-two stand-in N_t = 2^20
    # (Δt = 2^-20 ≈ 9.5e-7; reading R#24); u = u_xx = 0 (the c1 operator); the paper's
    # random start is read as noise on top of the c1 sine.
    "c6": Problem("c6", "biharmonic", "hinged", 1, m=64, nt=1 << 20, t_window=1.0, alpha=1e-3,
                  u0_kind="sine_plus_noise", u0_range=(-0.01, 0.01), seed=6),
    # NEXT-3 as the paper states it (Fig. 3 neighbourhood): 1D biharmonic with
    # the paper's Neumann Δ_h, h = 1/64 (65 nodes), Δt = 10⁻⁶, N_t = 10⁶ = 2⁶·5⁶
    # (the mixed-radix four-step time pass, k_tmix.cuh: 1000 × 1000), T = 1, α = 10⁻³
    "c6n": Problem("c6n", "biharmonic", "neumann", 1, m=64, nt=10 ** 6, t_window=1.0, alpha=1e-3,
                   u0_kind="sine_plus_noise", u0_range=(-0.01, 0.01), seed=6),
    # NEXT-4: c4's PinT-I with the paper's time-only averaged Jacobian
    # J̃ = I_t ⊗ (1/N_t) Σ_n J_s(u_n) — spatially varying, Step-(2) solved by an inner Krylov
    # iteration preconditioned by the scalar-J̄ spectral solve
    "c4t": Problem("c4t", "cahn_hilliard", "neumann", 2, m=256, nt=64, t_window=64e-4, alpha=1e-3,
                   eps=0.02, n_windows=4, max_iter=400, omega=0.7, tau=1.0,
                   u0_range=(-0.1, 0.1), seed=4, jacobian="time_avg"),
}


def config(name: str) -> Problem:
    return CONFIGS[name]


def twin(name: str, **kw) -> Problem:
    """Reduced twin: same physics, smaller grid / Nt (parity cases the oracle finishes in seconds)."""
    return replace(CONFIGS[name], name=name + "_twin", **kw)
