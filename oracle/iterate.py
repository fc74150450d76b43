"""All-at-once residuals and the ParaDiag outer iteration (ORACLE — test infrastructure only).

Linear: K = C1^(0)⊗I + C2^(0)⊗A, b = ((I/Δt - (1-θ)A) u0, 0, …, 0) (R#3).  The paper's
WR step P_α U^k = b^{k-1} is, algebraically, the defect correction
    U^k = U^{k-1} + P_α⁻¹ (b - K U^{k-1})
because b^{k-1} = b + (P_α - K) U^{k-1}.

Cahn-Hilliard PinT-I with one quasi-Newton step per WR step (R#6):
    U^k = U^{k-1} + ω_k P̃⁻¹ (-G(U^{k-1})),  -G(U)_n = -(U_n - U_{n-1})/Δt + Δ_h(U_n³ - U_n - ε²Δ_h U_n)
(P:460-463 with the α-terms cancelled as above), P̃ with the scalar J̄ = mean(3U² - 1) (R#7, R#8),
or (jacobian = "time_avg", NEXT-4) with the paper's time-only average J̃ = diag(mean_n 3U_n²),
ω_k = min(omega, tau/‖δ_k‖∞) (R#9; linear problems ω = 1).

Stopping (R#4): ‖δ^k‖∞ ≤ tol·‖U^k‖∞ with the undamped δ; c5 runs a fixed K (R#16).
Initial iterate (R#5): U⁰ = u0 broadcast, or U⁰ = 0.  Windows (R#19): u0 ← U_{N_t}.
"""
import numpy as np

from . import spatial, circulant, precond


def _shift_prev(u0: np.ndarray, U: np.ndarray) -> np.ndarray:
    """U_{n-1} for n = 1..N_t with U_0 := u0."""
    return np.concatenate([u0[None], U[:-1]], axis=0)


def residual_linear(prob, u0: np.ndarray, U: np.ndarray) -> np.ndarray:
    """r = b - K U, r_n = -(U_n - U_{n-1})/Δt - A(θ U_n + (1-θ) U_{n-1})."""
    Uprev = _shift_prev(u0, U)
    r = -(U - Uprev) * circulant.inv_dt(prob)
    if prob.theta == 1.0:
        return r - spatial.apply_A(U, prob)
    return r - (prob.theta * spatial.apply_A(U, prob) + (1.0 - prob.theta) * spatial.apply_A(Uprev, prob))


def residual_ch(prob, u0: np.ndarray, U: np.ndarray):
    """-G(U) of P:460-463 (mixed form v = f(u) - ε²Δ_h u) and J̄ = mean(3U² - 1)."""
    _, e2 = spatial.coeffs(prob)
    Uprev = _shift_prev(u0, U)
    v = U * U * U - U - e2 * spatial.lap(U, prob.m, prob.bc, prob.dim)
    r = spatial.lap(v, prob.m, prob.bc, prob.dim) - (U - Uprev) * circulant.inv_dt(prob)
    jbar = float(np.mean(3.0 * U * U - 1.0))
    return r, jbar


def residual_ch_eyre(prob, u0: np.ndarray, U: np.ndarray):
    """PinT-II (NEXT-1): Eyre's splitting treats the convex part u³ implicitly and the
    concave -u explicitly, u_n - u_{n-1} = Δt(Δ_h u_n³ - Δ_h u_{n-1} - ε²Δ_h² u_n).  The
    defect of the sequential scheme (= -Q(U) with the α-terms cancelled) in nested form:
        r_n = (Δ_h(U_n³ - ε²Δ_h U_n) - Δ_h U_{n-1}) - (U_n - U_{n-1})/Δt,   U_0 := u0,
    and the averaged Jacobian of the implicit part J̄₃ = mean(3U²) (R#8 reading of J̃)."""
    _, e2 = spatial.coeffs(prob)
    Uprev = _shift_prev(u0, U)
    v = U * U * U - e2 * spatial.lap(U, prob.m, prob.bc, prob.dim)
    r = (spatial.lap(v, prob.m, prob.bc, prob.dim) - spatial.lap(Uprev, prob.m, prob.bc, prob.dim)) - \
        (U - Uprev) * circulant.inv_dt(prob)
    jbar = float(np.mean(3.0 * U * U))
    return r, jbar


def is_ch(prob) -> bool:
    return prob.kind in ("cahn_hilliard", "cahn_hilliard_eyre")


def residual(prob, u0, U):
    if prob.kind == "cahn_hilliard":
        return residual_ch(prob, u0, U)
    if prob.kind == "cahn_hilliard_eyre":
        return residual_ch_eyre(prob, u0, U)
    return residual_linear(prob, u0, U), 0.0


def initial_iterate(prob, u0: np.ndarray) -> np.ndarray:
    shape = (prob.nt,) + (u0.shape if prob.dim == 2 else u0.shape[-1:])
    if prob.init == "zero":
        return np.zeros(shape)
    return np.broadcast_to(u0.reshape(shape[1:]), shape).copy()


def time_avg_jacobian(U: np.ndarray) -> np.ndarray:
    """jt = (1/N_t) Σ_n 3 u_n² per grid point: the diagonal of J̃ = (1/N_t) Σ_n J_s(u_n) (R#7)."""
    return 3.0 * np.mean(U * U, axis=0)


def iterate_once(prob, u0, U):
    """One ParaDiag iteration.  Returns (U_new, info dict)."""
    r, jbar = residual(prob, u0, U)
    jt = time_avg_jacobian(U) if is_ch(prob) and getattr(prob, "jacobian", "scalar") == "time_avg" else None
    delta, imag = precond.apply_precond(prob, r, jbar, jt)
    dmax = float(np.abs(delta).max())
    if is_ch(prob):
        omega = min(prob.omega, prob.tau / dmax) if dmax > 0 else prob.omega
    else:
        omega = prob.omega
    U_new = U + omega * delta
    umax = float(np.abs(U_new).max())
    return U_new, dict(delta_max=dmax, u_max=umax, rel=dmax / umax if umax > 0 else 0.0,
                       jbar=jbar, omega=omega, imag=imag)


GROWTH_LIMIT = 3   # ‖δ‖∞ growing in 3 consecutive iterations flags the window diverging


def solve_window(prob, u0, U=None, history=None, flags=None):
    """Iterate one window until the stop rule (or fixed K / max_iter).  Returns (U, iters, converged).

    Failure detection: when the undamped increment ‖δ_k‖∞ exceeds ‖δ_{k-1}‖∞ in
    GROWTH_LIMIT consecutive iterations the window is diverging (e.g. BJ.c5, outside Thm 3.3's
    hypothesis): it stops unconverged, or with fixed K is only flagged.  flags (a list)
    receives True/False per window."""
    u0 = np.asarray(u0, dtype=np.float64)
    if prob.dim == 1:
        u0 = u0.reshape(-1)
    if U is None:
        U = initial_iterate(prob, u0)
    kmax = prob.fixed_iters if prob.fixed_iters is not None else prob.max_iter
    converged = False
    k = 0
    growth, prev, diverging = 0, None, False
    for k in range(1, kmax + 1):
        U, info = iterate_once(prob, u0, U)
        if history is not None:
            history.append(info)
        if not np.isfinite(info["delta_max"]) or not np.isfinite(info["u_max"]):
            break
        if prob.fixed_iters is None and info["delta_max"] <= prob.tol * info["u_max"]:
            converged = True
            break
        growth = growth + 1 if prev is not None and info["delta_max"] > prev else 0
        prev = info["delta_max"]
        if growth >= GROWTH_LIMIT:
            diverging = True
            if prob.fixed_iters is None:
                break
    if flags is not None:
        flags.append(diverging)
    return U, k, converged


def solve(prob, u0, history=None, flags=None):
    """All windows.  Returns (U of the last window, [iters per window], [converged], [U_Nt per window])."""
    u0 = np.asarray(u0, dtype=np.float64)
    iters, conv, finals = [], [], []
    U = None
    for _ in range(prob.n_windows):
        U, k, c = solve_window(prob, u0, history=history, flags=flags)
        iters.append(k)
        conv.append(c)
        finals.append(U[-1].copy())
        u0 = U[-1].copy()
    return U, iters, conv, finals
