/*
 * paradiag.h — C ABI of the B200-native ParaDiag preconditioner library (libparadiag.so).
 *
 * Garai & Mandal, "Diagonalization Based Parallel-in-Time Method for a Class of Fourth Order
 * Time Dependent PDEs" (arXiv 2304.14021).  Citations "P:L" are lines of /root/reference/PAPER.md;
 * "R#n" are the readings listed in DESIGN.md §3.
 *
 * The hot path is the α-circulant preconditioner application δ = P_α⁻¹ r, the paper's three
 * steps (eq. pintiter1; CH PinT-I P:491-499, eq. pintiter_CH):
 *   Step-(1) scale by Γ_α = diag(α^{j/N_t}) and DFT along time for every spatial dof;
 *   Step-(2) N_t independent shifted spatial solves (d_l I + A) x = ŝ_l  (1D: pentadiagonal LU
 *            + one nested-residual refinement; 2D: DCT-I (Neumann) / DST-I (hinged) diagonalisation,
 *            CH: per-mode divide by d_l - J̄Λ + ε²Λ²);
 *   Step-(3) inverse DFT along time and unscale by Γ_α⁻¹.
 * plus the all-at-once residual r = b - K(U) and the defect-correction
 * update U ← U + ω δ that together form one ParaDiag iteration.
 *
 * Conventions for every entry point
 *  - Pointers named d_* / U / r / delta / u0 are CUDA DEVICE pointers to float64 arrays owned by
 *    the caller; the library owns only its internal workspace.  *_host entry points take HOST
 *    pointers instead (pageable or pinned).
 *  - Layout: U, r, delta are [nt][ny][nx] row-major contiguous (time slowest, x fastest), holding
 *    u_1..u_{N_t} (u_0 excluded, as the paper's U).  u0 is [ny][nx].  ny = 1 in 1D.
 *    Neumann unknowns include the boundary nodes (m+1 per axis); hinged (u = Δu = 0,
 *    P:703 case (ii)) unknowns are the interior nodes (m-1 per axis).  h = 1/m.
 *  - Work is enqueued on the stream passed to paradiag_init, in order.  apply_precond and
 *    residual are asynchronous; iterate / solve synchronise once per iteration on 4 scalars.
 *  - A handle must not be used from two host threads at once.
 *  - Return value: PD_OK (0), PD_NOT_CONVERGED (1, a status), or a negative error code;
 *    paradiag_strerror() names it and paradiag_last_error() gives a detail string for the
 *    calling thread.  No entry point falls back to a CPU path: without a usable sm_100a device
 *    they return PD_ECUDA.
 */
#ifndef PARADIAG_H
#define PARADIAG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARADIAG_ABI_VERSION 5

#if defined(__GNUC__)
#define PD_API __attribute__((visibility("default")))
#else
#define PD_API
#endif

/* return codes (SPEC-style error convention) */
#define PD_OK              0
#define PD_NOT_CONVERGED   1   /* status, not an error: non-convergence is a flag            */
#define PD_EINVAL        (-1)  /* invalid problem / argument                                  */
#define PD_ESINGULAR     (-2)  /* some shifted system d_l + e_l μ is (numerically) singular   */
#define PD_ECUDA         (-3)  /* CUDA runtime failure (incl. no device / wrong arch)          */
#define PD_ENCCL         (-4)  /* reserved: multi-GPU communicator failure                     */
#define PD_ENOMEM        (-5)  /* device allocation failed                                     */
#define PD_EDIVERGED     (-6)  /* non-finite iterate / increment                               */

/* problem kinds */
#define PD_BIHARMONIC      0   /* u_t = -Δ²u                      A = Δ_h²  */
#define PD_LINEAR_CH       1   /* u_t = -β²Δu - ε²Δ²u             A = β²Δ_h + ε²Δ_h²  */
#define PD_CAHN_HILLIARD   2   /* u_t = Δ(u³ - u - ε²Δu), PinT-I           */
#define PD_CAHN_HILLIARD_EYRE 3 /* same PDE, PinT-II: Eyre convex splitting, u³ implicit, -u lagged
                                   (P:502-545); Step-(2) divisor d_l + λ_{3,l}Λ - J̄₃Λ + ε²Λ²,
                                   J̄₃ = mean(3U²)                                                */

/* boundary conditions */
#define PD_BC_NEUMANN      0   /* ∂u = ∂Δu = 0, paper Δ_h with ghost reflection */
#define PD_BC_HINGED       1   /* u = Δu = 0 (P:703 case (ii)), zero ghosts at each Δ_h (R#14)  */

/* initial iterate U⁰ (R#5) */
#define PD_INIT_BROADCAST  0   /* U⁰_n = u0 for every n */
#define PD_INIT_ZERO       1   /* U⁰ = 0                */
#define PD_JACOBIAN_SCALAR   0 /* CH Step-(2): scalar J̄ (R#8), one spectral solve          */
#define PD_JACOBIAN_TIME_AVG 1 /* CH Step-(2): J̃ = diag(mean_n 3U_n²), inner GMRES */

typedef struct pd_problem {
  int32_t kind;          /* PD_BIHARMONIC | PD_LINEAR_CH | PD_CAHN_HILLIARD | PD_CAHN_HILLIARD_EYRE */
  int32_t bc;            /* PD_BC_NEUMANN | PD_BC_HINGED (CH: Neumann only)                */
  int32_t dim;           /* 1 or 2 (CH: 2 only)                                                  */
  int32_t nt;            /* time steps per window, power of two in [2, 2^20] (> 4096: k_tlong.cuh) */
  int64_t m;             /* intervals per axis, h = 1/m; 2D: power of two in [4, 4096]; 1D ≥ 4   */
  double  t_window;      /* window length T; Δt = T / nt, 1/Δt evaluated as nt / T (R#20)        */
  double  alpha;         /* PinT parameter α ∈ (0, 1)                              */
  double  theta;         /* θ-method parameter in [1/2, 1]; CH: 1 (backward Euler)   */
  double  beta;          /* LINEAR_CH β; β² := fl(β·β)                                     */
  double  eps;           /* LINEAR_CH / CH ε ≥ 0; ε² := fl(ε·ε)                                   */
  double  tol;           /* stop when ‖δ‖∞ ≤ tol·‖U‖∞ (R#4)                                       */
  double  omega;         /* damping cap: ω_k = min(omega, tau/‖δ_k‖∞) for CH (R#9); linear ω = 1 */
  double  tau;
  int32_t n_windows;     /* sequential windows, u0 ← U_{N_t} between them                */
  int32_t max_iter;      /* iteration cap per window                                              */
  int32_t fixed_iters;   /* > 0: run exactly this many iterations per window, no stop test (c5)  */
  int32_t init;          /* PD_INIT_BROADCAST | PD_INIT_ZERO                                      */
  int32_t jacobian;      /* CH Step-(2) Jacobian: PD_JACOBIAN_SCALAR (J̄ = mean(3U²-1), R#8) or
                            PD_JACOBIAN_TIME_AVG (J̃ = diag(mean_n 3U_n²), NEXT-4: inner
                            GMRES preconditioned by the scalar solve); linear kinds: 0          */
  int32_t reserved;      /* 0                                                                     */
} pd_problem;

typedef struct pd_handle pd_handle;

typedef struct pd_iter_info {
  int32_t iters;         /* iterations done in the current window after this call                */
  int32_t converged;     /* ‖δ‖∞ ≤ tol·‖U‖∞ reached                                               */
  double  delta_max;     /* ‖δ_k‖∞ (undamped increment)                                           */
  double  u_max;         /* ‖U^k‖∞ after the update                                               */
  double  rel;           /* delta_max / u_max                                                     */
  double  jbar;          /* J̄ = mean(3U²-1) used by the CH preconditioner (0 for linear)          */
  double  omega;         /* damping factor applied                                                */
  int32_t growth;        /* consecutive iterations (this window) with ‖δ_k‖∞ > ‖δ_{k-1}‖∞; at
                            PD_GROWTH_LIMIT the window is flagged diverging          */
} pd_iter_info;

/* Divergence flag (SURVEY §5.3 failure detection): a window whose undamped increment ‖δ‖∞ grew in
 * PD_GROWTH_LIMIT consecutive iterations is diverging — e.g. BJ.c5, which violates the hypothesis
 * of Thm 3.3.  paradiag_solve stops such a window with PD_NOT_CONVERGED (fixed_iters
 * runs keep iterating and only flag it).  The oracle applies the same rule (oracle/iterate.py). */
#define PD_GROWTH_LIMIT 3

#define PD_MAX_WINDOWS 64
typedef struct pd_solve_info {
  int32_t windows_done;
  int32_t converged;     /* all windows converged (fixed_iters > 0: always 0)                      */
  int32_t iters[PD_MAX_WINDOWS];
  double  last_rel[PD_MAX_WINDOWS];
  double  seconds;       /* host wall time of the call                                             */
  int32_t diverging;     /* windows flagged diverging (PD_GROWTH_LIMIT rule, see pd_iter_info)      */
} pd_solve_info;

/* ABI version (PARADIAG_ABI_VERSION); lets a binding check it loaded the library it expects. */
PD_API int paradiag_abi_version(void);

/* Name of a return code; never NULL. */
PD_API const char* paradiag_strerror(int code);

/* Detail message of the last failing call on this host thread ("" if none). */
PD_API const char* paradiag_last_error(void);

/* Device workspace the handle will allocate for `p` (bytes, excluding the caller's U/r/δ), per
 * rank when nranks > 1.  Returns PD_EINVAL if the problem is not supported. */
PD_API int paradiag_workspace_bytes(const pd_problem* p, int nranks, size_t* bytes);

/* Create a handle on CUDA device `device`, enqueuing on `cuda_stream` (a cudaStream_t; NULL =
 * legacy default stream).  Validates the problem (PD_EINVAL), checks the shifted systems for
 * singularity (PD_ESINGULAR), builds the Γ_α / d_l / Λ / twiddle tables and, in 1D, factorises
 * the N_t/2+1 pentadiagonal matrices d_l I + A (no pivoting).  On success *out owns all workspace.
 *
 * Multi-GPU (one process per GPU): with nccl_id != NULL the handle
 * is rank `rank` of `nranks` (≤ 8) of a slab-sharded 2D linear problem (θ = 1, the register-FFT
 * sizes 64 ≤ m ≤ 2048, 32 ≤ N_t ≤ 1024; "Step-(2) is fully parallel").  The library creates
 * and owns the NCCL communicator (ncclCommInitRank with the NCCL the process has loaded — torch's)
 * and runs the halo exchange, the two all-to-all transposes per P_α⁻¹ and the max all-reduce of
 * the stop rule itself; the caller passes only its row slab (paradiag_local_rows): u0 [ny_l][nx],
 * U / r / δ [nt][ny_l][nx].  Every rank must make the same calls in the same order; an id serves
 * one communicator (draw a fresh one per sharded handle).
 * nccl_id = NULL and nranks ≤ 1: a single-GPU handle (rank ignored). */
PD_API int paradiag_init(const pd_problem* p, int device, void* cuda_stream, const unsigned char* nccl_id,
                         int rank, int nranks, pd_handle** out);

/* A fresh NCCL unique id (128 bytes) for paradiag_init: call on rank 0 only and broadcast it (e.g.
 * with torch.distributed).  PD_ENCCL if NCCL cannot be resolved (import torch first). */
PD_API int paradiag_nccl_unique_id(unsigned char id[128]);

/* The rows [y0, y0 + ny_local) of the grid this handle's rank owns (single GPU: 0 and ny). */
PD_API int paradiag_local_rows(const pd_handle* h, int64_t* y0, int64_t* ny_local);

/* Verification hook of the sharded engine without a multi-GPU box: nranks VIRTUAL ranks in one
 * process on one device (out[nranks] receives their handles), driven phase by phase in rank order
 * with the collectives emulated by device copies — no rank ever waits on another.  Same layouts and
 * kernels as the NCCL path; iterate / solve take the ranks' row-slab pointers in rank order.
 * Destroy every handle with paradiag_destroy. */
PD_API int paradiag_init_virtual(const pd_problem* p, int device, void* cuda_stream, int nranks, pd_handle** out);
PD_API int paradiag_iterate_virtual(pd_handle* const* hs, int nranks, const double* const* u0_l,
                                    double* const* U_l, pd_iter_info* info);
PD_API int paradiag_solve_virtual(pd_handle* const* hs, int nranks, const double* const* u0_l,
                                  double* const* U_l, pd_solve_info* info);

/* The slab layout the sharded engine uses for rank `rank` of `nranks` on an n × n grid with nt
 * slices (host only, no CUDA): out = {y0, ny_l, x0, nx_l, nsr, so, fs[P], fr[P], cfs[P], cfr[P],
 * then the four transpose-block maps x_out, y_in, y_out, x_in, each {P, (e0, cnt, off) × P}};
 * fs / fr = forward send / receive element counts per peer (0 for the rank itself), cfs / cfr their
 * offsets in the send [0, nsr) / receive [nsr, 2 nsr) regions, so = the kept block.  cap = capacity
 * of out (≥ 6 + 4P + 4(1 + 3P)).  Lets the CPU tests check the engine's maps. */
PD_API int paradiag_shard_layout(int64_t n, int64_t nt, int nranks, int rank, int64_t* out, int64_t cap);

/* Residual r = b - K(U) of the all-at-once system (P:127-149 linear; -G(U) of P:460-463 for CH,
 * mixed form v = U³ - U - ε²Δ_h U, r = Δ_h v - (U_n - U_{n-1})/Δt), with U_0 := u0, stencils in
 * nested form (R#15).  For CH also reduces J̄ = mean(3U² - 1) into the handle (device-resident),
 * which the next paradiag_apply_precond_dev-style use (iterate) consumes.  r must not alias U.
 * If jbar_out != NULL the call synchronises and stores J̄ there (0 for linear kinds). */
PD_API int paradiag_residual(pd_handle* h, const double* u0, const double* U, double* r, double* jbar_out);

/* δ = P_α⁻¹ r — Steps (1)-(3), P:158-169 / P:491-499.  `jbar` is the scalar Jacobian average used
 * by CH (ignored otherwise).  r and delta may alias (in-place).  Asynchronous. */
PD_API int paradiag_apply_precond(pd_handle* h, const double* r, double* delta, double jbar);

/* δ = G̃'⁻¹ r with the time-only averaged Jacobian J̃ = diag(jt) of P:486 (NEXT-4; CH kinds, 2D,
 * jacobian = PD_JACOBIAN_TIME_AVG): jt [ny][nx] (device) is the per-point time mean of 3U², so
 * Step-(2) of P:495 (PinT-I) / P:545 (PinT-II) is (λ_{1,l} I - Δ_h diag(jt) + {1, λ_{3,l}} Δ_h +
 * ε²Δ_h²) per bin.  Solved in the time domain as G̃' δ = r by restarted GMRES, left-preconditioned
 * by the scalar-J̄ P_α⁻¹ with J̄ = mean(jt) - {1, 0}, to a relative preconditioned residual of
 * 1e-13.  r and delta may alias.  Synchronises (one host read per Krylov step).
 * PD_NOT_CONVERGED if the inner solve hit its iteration cap. */
PD_API int paradiag_apply_precond_jt(pd_handle* h, const double* r, double* delta, const double* jt);

/* One ParaDiag iteration on window data: r = b - K(U) (or -G(U)), δ = P_α⁻¹ r, U ← U + ω δ, with
 * ω = 1 (linear) or min(omega, tau/‖δ‖∞) (CH, R#9).  Fills *info (synchronises on 4 scalars).
 * Returns PD_EDIVERGED if a non-finite value appeared. */
PD_API int paradiag_iterate(pd_handle* h, const double* u0, double* U, pd_iter_info* info);

/* Full solve: for each window, set U⁰ (broadcast or zero), iterate until ‖δ‖∞ ≤ tol‖U‖∞ (or
 * exactly fixed_iters times), then hand u_{N_t} to the next window.  u0 is not modified;
 * on return U holds the last window's iterate.  PD_NOT_CONVERGED if a window hit max_iter or was
 * stopped as diverging (info->diverging counts the flagged windows; PD_GROWTH_LIMIT). */
PD_API int paradiag_solve(pd_handle* h, const double* u0, double* U, pd_solve_info* info);

/* As paradiag_solve but with HOST buffers: copies u0_host ([ny][nx]) to the device, solves into
 * a library-owned U, and copies the final time slice u_{N_t} of the last window to uT_host
 * ([ny][nx]).  The copies are part of the call (end-to-end path). */
PD_API int paradiag_solve_host(pd_handle* h, const double* u0_host, double* uT_host, pd_solve_info* info);

/* Number of kernel launches one paradiag_iterate enqueues (for launch accounting); -1 when it is
 * data dependent (jacobian = PD_JACOBIAN_TIME_AVG: inner GMRES steps). */
PD_API int paradiag_launches_per_iteration(const pd_handle* h);

/* Per-kernel device time, measured with CUDA events recorded around each launch on the
 * handle's stream during paradiag_iterate / paradiag_solve (enable with paradiag_profile). */
typedef struct pd_kernel_time {
  char    name[32];
  int32_t launches;
  double  total_ms;
} pd_kernel_time;

/* Enable (1) / disable (0) per-kernel event timing and reset the accumulators. */
PD_API int paradiag_profile(pd_handle* h, int enable);

/* Copy up to max_entries accumulated kernel timings into out; *n_out = entries available. */
PD_API int paradiag_profile_read(const pd_handle* h, pd_kernel_time* out, int max_entries, int* n_out);

/* ---------------------------------------------------------------------------------------------
 * Multi-rank (slab) mode — SURVEY §8(e), DESIGN.md §8.  "Step-(2) is fully parallel" and
 * Steps (1)/(3) are independent per spatial point, so a 2D problem shards over P ranks (one process
 * per GPU): rank r owns the ROW slab y ∈ [y0, y0+nyl) of every time slice for the residual, the
 * x-direction transforms and the update, and the COLUMN slab x ∈ [x0, x0+nxl) (x-modes after the
 * x transform) for the y-direction transforms and the time pass (Γ_α·DFT, per-mode divide, IDFT,
 * Γ_α⁻¹).  Between the two layouts the caller runs an all-to-all transpose (torch.distributed /
 * NCCL); the 2-row residual halo is exchanged with the neighbouring ranks.  The per-rank entry
 * points below run only the local kernels; paper_2304_14021_b200/dist.py composes them.
 * Buffers (all device, fp64, caller-owned):
 *   u0_l [nyl][n], U_l / r_l / rows [nt][nyl][n]    row slab  (n = points per axis)
 *   halo_lo / halo_hi [nt][2][n]                     global rows y0-2, y0-1 / y0+nyl, y0+nyl+1
 *                                                    (NULL where the slab touches the boundary)
 *   cols [nt][n][nxl]                                column slab (row stride nxl)
 * Supported: 2D linear kinds (biharmonic, linearised CH), 64 <= m <= 2048, 32 <= nt <= 1024;
 * otherwise PD_EINVAL.  nyl >= 3.
 * ------------------------------------------------------------------------------------------- */
PD_API int paradiag_init_slab(const pd_problem* p, int device, void* cuda_stream, int64_t y0, int64_t nyl,
                              int64_t x0, int64_t nxl, pd_handle** out);
PD_API int paradiag_slab_geometry(const pd_handle* h, int64_t* y0, int64_t* nyl, int64_t* x0, int64_t* nxl);
/* r_l = b - K(U) on the row slab (nested stencils R#15), halos as above. */
PD_API int paradiag_slab_residual(pd_handle* h, const double* u0_l, const double* U_l, const double* halo_lo,
                                  const double* halo_hi, double* r_l);
/* DCT-I / DST-I along x of every local row; want_dmax: fold max|out| into the
 * handle's ‖δ‖∞ statistic (the inverse pass).  in may alias out. */
PD_API int paradiag_slab_xpass(pd_handle* h, const double* in, double* out, int want_dmax);
/* In place on the column slab: y transform, time pass (Steps (1)-(3) per spatial mode),
 * inverse y transform. */
PD_API int paradiag_slab_ypass(pd_handle* h, double* cols);
/* The same passes reading / writing the all-to-all buffers directly (no pack / unpack copies):
 * seg_* = NULL means the slab layout above; otherwise an int64 host array {k, (e0, cnt, off) × k}
 * (k ≤ 8, blocks tiling the line in order) describing transpose blocks:
 *   x pass (lines along x, local line ln = n·nyl + y): element x ∈ [e0_q, e0_q + cnt_q) lives at
 *     buf[off_q + ln·cnt_q + (x − e0_q)]   (block q = [nt][nyl][cnt_q], the send/recv block of peer q)
 *   y pass (lines along y): row y ∈ [e0_s, e0_s + cnt_s) of slice n, local column c lives at
 *     buf[off_s + (n·cnt_s + y − e0_s)·nxl + c]   (block s = [nt][cnt_s][nxl])
 * slab_ypass_seg runs y-DTT (in → cols), the time pass in place on cols, y-DTT⁻¹ (cols → out).
 * in must not alias out unless both are the slab (seg NULL). */
PD_API int paradiag_slab_xpass_seg(pd_handle* h, const double* in, double* out, int want_dmax,
                                   const int64_t* seg_in, const int64_t* seg_out);
PD_API int paradiag_slab_ypass_seg(pd_handle* h, const double* in, double* cols, double* out,
                                   const int64_t* seg_in, const int64_t* seg_out);
/* Slice-range forms for overlapping the all-to-all with the passes (slices [n0, n0 + nn)):
 * slab-layout buffers (seg NULL) are given from slice 0 and shifted by the library; block buffers
 * are addressed relative to the range (the map's offsets point at this range's blocks, each
 * [nn][…][cnt] / [nn][cnt][nxl]).  yrange stage 0: y-DTT in → cols, 1: the time pass on cols (all
 * slices, n0/nn ignored), 2: y-DTT⁻¹ cols → out. */
PD_API int paradiag_slab_xrange(pd_handle* h, const double* in, double* out, int want_dmax,
                                const int64_t* seg_in, const int64_t* seg_out, int64_t n0, int64_t nn);
PD_API int paradiag_slab_yrange(pd_handle* h, const double* in, double* cols, double* out, int stage,
                                const int64_t* seg, int64_t n0, int64_t nn);
PD_API int paradiag_slab_update_range(pd_handle* h, double* U_l, const double* delta_l, int64_t n0, int64_t nn);
/* Peer-memory transposes (opt-in): a block map offset may point into another rank's
 * buffer mapped into this process (element offset from the call's buffer pointer, possibly
 * negative), so the x pass and the inverse y pass store their peer blocks straight into the peers'
 * receive buffers over NVLink.  These wrap CUDA IPC: export a device allocation (64-byte handle),
 * map a peer's, unmap. */
PD_API int paradiag_ipc_handle(const void* dev_ptr, unsigned char handle[64]);
PD_API int paradiag_ipc_open(const unsigned char handle[64], void** dev_ptr);
PD_API int paradiag_ipc_close(void* dev_ptr);
/* U_l += δ_l (ω = 1) and fold max|U| into the handle's ‖U‖∞ statistic. */
PD_API int paradiag_slab_update(pd_handle* h, double* U_l, const double* delta_l);
/* dst[a*d0 + b*d1 + c] = src[a*s0 + b*s1 + c], a < n0, b < n1, c < n2 (element strides): the pack /
 * unpack of the transposes.  Any handle (its stream is used). */
PD_API int paradiag_copy3d(pd_handle* h, const double* src, double* dst, int64_t n0, int64_t n1, int64_t n2,
                           int64_t s0, int64_t s1, int64_t d0, int64_t d1);
/* ---------------------------------------------------------------------------------------------
 * Time slabs — 1D long windows across ranks (SURVEY §8(f) NEXT-3 "frequency sharding with a tiny
 * spatial problem").  Steps (1)/(3) are per spatial mode and Step (2) per time bin
 * (P:158-169), the residual couples only u_n and u_{n-1}.  Every rank holds a handle of
 * the GLOBAL problem (paradiag_init; 1D linear kind, N_t > 4096 or PARADIAG_TLONG, N_x <= 64) and
 * owns the contiguous time rows [n0, n0 + nn) of U for the residual, the x transforms and the
 * update, and the column block [c0, c0 + bcols) of x-modes (all N_t rows) for the time pass.
 * Between the two an all-to-all moves the blocks (dist.py, TimeSlabRank).
 * Layouts (device, fp64, caller-owned):
 *   u_prev [N_x]          the row before n0: u0 for n0 = 0, else the previous rank's last row
 *   U_l [nn][N_x]         the rank's rows
 *   blocks [pitch/bcols][nn][bcols]   r̂ / δ̂ of the rank's rows, block q = x-modes [q·bcols, ...)
 *                                     (block q is the all-to-all chunk of rank q)
 *   cols [N_t][bcols]     the x-modes [c0, c0 + bcols) of every time row
 * pitch = 2⌈N_x/2⌉ (paradiag_tslab_pitch); bcols even, dividing pitch; modes past N_x are padding.
 * paradiag_tslab_residual: blocks = T·(b − K U) of the rows (nested stencils R#15).
 * paradiag_tslab_time: in place Γ_α-scaled DFT, divide per bin and mode, inverse on the
 *   column block (a block of padding only is a no-op).
 * paradiag_tslab_update: δ = T·δ̂ from blocks, U_l += δ, fold ‖δ‖∞ / ‖U‖∞ of the rows into the handle's
 *   statistics (reset / read below; the caller reduces them over ranks).
 * Errors: PD_EINVAL for another kind of handle, bad bcols / c0 / nn, NULL buffers. */
PD_API int paradiag_tslab_pitch(const pd_handle* h, int64_t* pitch);
PD_API int paradiag_tslab_residual(pd_handle* h, const double* u_prev, const double* U_l, int64_t nn, double* blocks,
                                   int64_t bcols);
PD_API int paradiag_tslab_time(pd_handle* h, double* cols, int64_t c0, int64_t bcols);
PD_API int paradiag_tslab_update(pd_handle* h, const double* blocks, int64_t bcols, double* U_l, int64_t nn);

/* Zero the handle's ‖δ‖∞ / ‖U‖∞ statistics (asynchronous) / read them (synchronises the stream). */
PD_API int paradiag_stats_reset(pd_handle* h);
PD_API int paradiag_stats_read(pd_handle* h, double* dmax, double* umax);

/* Release all device memory of the handle.  NULL is a no-op. */
PD_API void paradiag_destroy(pd_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* PARADIAG_H */
