// paradiag.cu — C ABI (include/paradiag.h) and the single-GPU iteration engine.
//
// One ParaDiag iteration = residual (P:127-149 / P:452-463) → P_α⁻¹ (P:158-169 / P:491-499) →
// update U ← U + ω δ.  2D pass order (spatial-first):
//   x-DTT (r → δ) · y-DTT · fused time pass (Γ_α·DFT · per-mode divide · IDFT·Γ_α⁻¹) · y-DTT · x-DTT
// 1D: time DFT → batched pentadiagonal solves per bin → inverse time DFT.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <new>
#include <string>
#include <vector>

#include "../../include/paradiag.h"
#include "common.cuh"
#include "fft.cuh"
#include "k_misc.cuh"
#include "k_penta.cuh"
#include "k_residual.cuh"
#include "k_spatial.cuh"
#include "k_time.cuh"
#include "fast_launch.cuh"
#include "tlong.h"
#include "k_x1d.cuh"
#include "k_krylov.cuh"
#include "shard.h"

using namespace pd;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define PD_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(e_ == cudaErrorMemoryAllocation ? PD_ENOMEM : PD_ECUDA,               \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                  \
  } while (0)

#define PD_LAUNCHED()                                                                   \
  do {                                                                                  \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess)                                                              \
      return fail(PD_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_));   \
  } while (0)

enum KernelId { K_RESET = 0, K_RESIDUAL, K_JBAR, K_XFWD, K_YFWD, K_TIME, K_YINV, K_XINV, K_UPDATE,
                K_TFWD1D, K_PENTA, K_TINV1D, K_XINVUPD, K_RESUPD, K_TLA, K_TLB, K_TLD, K_TLBI, K_TLAI,
                K_XRES, K_XUPD, K_TLBF, K_KLAP, K_KVEC, PD_NKERNELS };
const char* kKernelNames[PD_NKERNELS] = {"reset_stats", "residual", "jbar_finalize", "dtt_x_fwd", "dtt_y_fwd",
                                         "time_solve_2d", "dtt_y_inv", "dtt_x_inv", "update",
                                         "time_fwd_1d", "penta_solve", "time_inv_1d", "dtt_x_inv_update",
                                         "residual_update", "tlong_a_fwd", "tlong_b_fwd", "tlong_divide",
                                         "tlong_b_inv", "tlong_a_inv", "residual_dst_x", "dst_x_inv_update",
                                         "tlong_b_fused", "krylov_lap_w", "krylov_vector_ops"};

constexpr int kTimeWarps = 8;   // 2D time pass: 16 spatial points (128-byte rows) per CTA
constexpr size_t kSmemMax = 227 * 1024;   // opt-in dynamic shared memory per CTA (sm_100a)
constexpr int kMaxNtShort = 4096;         // one pencil per warp on chip; longer windows: k_tlong.cuh
constexpr int kMaxNt = 1 << 20;           // four-step factors N1, N2 <= 1024
constexpr int kTime1DWarps = 4;
constexpr int kLineWarps = 4;   // spatial DTT rows: one warp per row, 4 rows per CTA
#ifndef PD_COLW
#define PD_COLW 8
#endif
constexpr int kColW = PD_COLW;  // spatial DTT columns: adjacent columns per CTA (one warp each)

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

// 2D tensor map of an [outer][pitch] fp64 array (inner extent `inner` <= pitch), boxes {box_w,
// box_h}, SWIZZLE_128B, 256-byte L2 promotion (measured faster than none for 128-byte box rows even
// though it over-reads when the neighbouring row segment is not used soon, ncu r02h).  The encoder is the driver's cuTensorMapEncodeTiled, resolved through the
// runtime (no -lcuda).  TMA needs 16-byte aligned rows: pitch even (tma.cuh).
bool make_map_2d(CUtensorMap* m, const double* base, int64_t inner, int64_t outer, int64_t pitch, unsigned box_w,
                 unsigned box_h) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !enc) {
      enc = nullptr;
      return false;
    }
  }
  if (reinterpret_cast<uintptr_t>(base) % 16 || (pitch & 1) || box_h > 256 || box_w * 8 > 128) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)(pitch * 8)};
  const cuuint32_t box[2] = {box_w, box_h};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// 3D tensor map of an [nt][ny][pitch] fp64 array (inner extent nx <= pitch, pitch even), boxes
// {box_w, box_h, 1}, no swizzle (the y⁻¹ staging chunks are plain [rows][8] tiles)
bool make_map_3d(CUtensorMap* m, const double* base, int64_t nx, int64_t ny, int64_t nt, int64_t pitch, unsigned box_w,
                 unsigned box_h) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !enc)
    return false;
  if (reinterpret_cast<uintptr_t>(base) % 16 || (pitch & 1) || box_h > 256) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nt};
  const cuuint64_t strides[2] = {(cuuint64_t)(pitch * 8), (cuuint64_t)(pitch * ny * 8)};
  const cuuint32_t box[3] = {box_w, box_h, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
int ilog2(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

}  // namespace

struct pd_handle {
  pd_problem P{};
  pd_shard* shard = nullptr;          // multi-rank slab sharding (shard.cu), NULL on a single-GPU handle
  int device = 0;
  cudaStream_t stream = nullptr;
  int nx = 0, ny = 0;
  int64_t ns = 0, total = 0;
  int log2nt = 0, log2h = 0, twlog = 0, nb = 0;
  bool neumann = true;
  bool fast = true;                   // register-FFT kernels (k_fast.cuh) where sizes allow
  bool tma = true;                    // PARADIAG_TMA=0: cp.async-staged time pass instead of TMA (A/B)
  // TMA time pass (k_time2d_v4): second workspace wt [nt][nx][lp], each slice COLUMN-MAJOR with the
  // line pitch lp = ny rounded up to even (k_cols_cm); the forward y pass writes it, the time pass
  // runs in place on it, the inverse y pass reads it
  double* wt = nullptr;
  int64_t ps = 0, lp = 0;             // wt slice pitch (nx·lp) and column-major line pitch
  // padded natural-layout workspace wp [nt][ny][lpx] between the x and y passes (M = 2048): row
  // pitch lpx = N_x rounded up to 8 doubles (64-byte aligned rows), so the inverse y pass stores
  // its tiles with TMA (k_cols_tma_inv, tensor map wp_map); PARADIAG_WP=0 turns it off (A/B)
  double* wp = nullptr;
  int64_t lpx = 0;
  CUtensorMap wp_map;
  double inv_dt = 0, inv_h2 = 0, b2 = 0, e2 = 0;
  // device buffers
  double* work = nullptr;             // 2D: δ/r workspace [nt][ns]; 1D: r [nt][nx]
  double2* spec = nullptr;            // 1D spectra [nx][nb] and scratch
  double2* w1 = nullptr;
  double2* w2 = nullptr;
  double* gam = nullptr;
  double* ginv = nullptr;
  double2* dl = nullptr;
  double2* el = nullptr;              // e_l = θ + (1-θ) z ω^l (NULL for θ = 1)
  double2* l3 = nullptr;              // λ_{3,l} = z ω^l (PinT-II only)
  double* lam = nullptr;
  double2* tw = nullptr;
  double2* trig = nullptr;
  double2* trig2 = nullptr;          // (cos, sin)(2πk/M) in the [j][b] layout of k_dtt.cuh
  double2* trigsc = nullptr;         // k_dtt.cuh pre-processing pairs: [M/2] sin, then [M/2] cos
  double2* trig2p = nullptr;         // (cos, sin)(2πk/M) in the [j][t] layout of k_dttp.cuh (M = 2048)
  // line kernels: 3 = k_dtt.cuh (default), 4 = k_dttp.cuh warp pairs for M = 2048 (opt-in: ncu d5b shows
  // it shared-memory bound, 12.2 vs 10.6 ms)
  int dtt_ver = 3;
  int tune = 0;                       // PARADIAG_TUNE: A/B switches for measurements
  int stagger_ns = 0;                 // PARADIAG_STAGGER: phase offset of co-resident CTAs (ns)
  // slab mode (multi-rank): rows [y0, y0+nyl) for residual / x passes / update,
  // columns [x0, x0+nxl) for the y passes and the time pass; buffers are the caller's
  bool slab = false;
  int y0 = 0, nyl = 0, x0 = 0, nxl = 0;
  double* band = nullptr;
  double2* fac = nullptr;             // 4 x [nx][nb]
  DevStats* st = nullptr;
  DevStats* st_host = nullptr;        // pinned
  double* jpart = nullptr;
  size_t njpart = 0;
  double* u0buf = nullptr;
  double* Uint = nullptr;             // solve_host's iterate
  // pipelined solve (linear 2D): iteration k's update U += δ is applied inside iteration k+1's
  // residual, which writes the new iterate to the other U buffer and r to the other workspace
  double* Ub = nullptr;
  double* work2 = nullptr;
  bool pipe = false;                  // PARADIAG_PIPELINE=1 enables (≈ neutral on c5, +2 arrays)
  // long windows (N_t > 4096, or PARADIAG_TLONG=1 from N_t = 1024): four-step time pass over HBM
  // (k_tlong.cuh); Y = spec, X = w1, each [N_t][⌈N_s/2⌉] complex.  1D then solves Step (2) in the
  // DST-I/DCT-I eigenbasis like 2D (x passes + per-mode divide) instead of the pentadiagonal LU.
  bool tlong = false;
  int log2n1 = 0, log2n2 = 0;
  int n1 = 0, n2 = 0;                 // N_t = n1·n2 (four-step factors)
  bool mixed = false;                 // N_t = 2^a 5^b, not a power of two: k_tmix.cuh passes
  int nst1 = 0, nst2 = 0;
  int8_t plan1[12] = {}, plan2[12] = {};
  double2* mtab = nullptr;            // mixed roots: W_{n1}^j (n1), W_{n2}^j (n2), W_N^b (b < n2)
  int* mrev = nullptr;                // digit reversals: rev1 [n1], irev1 [n1], rev2 [n2], irev2 [n2]
  // 1D long windows with N_x ≤ 64: x transforms as DMMA products with T (k_x1d.cuh), fused with
  // the residual (forward) and the update (inverse); x1T = Tᵀ zero padded to 64×64
  bool x1 = false;
  int mxp = 4;                        // PARADIAG_MXPAIRS: pencil pairs per CTA of the mixed-radix passes (4: two CTAs per SM, measured 3.49 vs 3.59 ms on c6n; or 8)
  bool tlfuse = true;                 // PARADIAG_TLFUSE=0: unfused pass B / divide / pass B⁻¹ (A/B, tests)
  double* x1T = nullptr;
  double* tlg = nullptr;              // k_tlong.cuh split Γ_α tables: ghi[N1] glo[N2] gihi[N1] gilo[N2]
  // NEXT-4 (jacobian = PD_JACOBIAN_TIME_AVG, k_krylov.cuh): jt = mean_n 3U², w' = jt - c - J̄,
  // GMRES(kKryM) basis V [kKryM+1][total], preconditioned right-hand side kb, dot partials
  double* jt = nullptr;
  double* wfld = nullptr;
  double* kV = nullptr;
  double* kb = nullptr;
  double* kpart = nullptr;
  double* kdev = nullptr;             // device copy of dot results / combination coefficients
  double* khost = nullptr;            // pinned
  int kry_last = 0;                   // Krylov steps of the last inner solve
  // device-side Arnoldi loop (k_krylov.cuh): state, its pinned mirror, K's fixed in/out vectors and
  // the WHILE graph of one cycle's steps; PARADIAG_KRYGRAPH=0 keeps the host loop (A/B, tests)
  bool kry_graph = true;
  KryDev* kd = nullptr;
  KryDev* kd_host = nullptr;
  double* kin = nullptr;
  double* kout = nullptr;
  cudaGraph_t kgraph = nullptr;
  cudaGraphExec_t kgexec = nullptr;
  cudaGraphConditionalHandle kcond;
  // Gram-Schmidt passes per Arnoldi step: 1 (measured c4t 3.3 s vs 4.7 s with 2, same counts and
  // parity; convergence is only ever declared on the recomputed true residual); PARADIAG_CGS_PASSES=2
  int cgs_passes = 1;
  bool penta_cta = true;              // PARADIAG_PENTA=0: the thread-per-bin pentadiagonal kernel
  int penta_refine = kPentaRefine;    // PARADIAG_PENTA_REFINE: refinement cap (A/B only)
  // device-side window loop (paradiag_solve): graph of a conditional WHILE node around one
  // iteration, captured for one U pointer; PARADIAG_GRAPH=0 keeps the host loop
  bool use_graph = true;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaGraphConditionalHandle gcond = 0;
  cudaStream_t cap_stream = nullptr;
  double* gU = nullptr;
  void* ctl = nullptr;                // LoopCtl (device)
  void* ctl_host = nullptr;           // pinned
  std::vector<void*> allocs;
  // optional per-kernel timing with CUDA events on the handle's stream (paradiag_profile)
  bool prof = false;
  cudaEvent_t ev[PD_NKERNELS][2] = {};
  bool ev_used[PD_NKERNELS] = {};
  double prof_ms[PD_NKERNELS] = {};
  int prof_n[PD_NKERNELS] = {};
};

namespace {

// Every pass is an NVTX range (header-only NVTX3: a no-op unless a tool such as ncu
// or nsys is attached) and, with paradiag_profile on, a pair of CUDA events.
void prof_begin(pd_handle* h, int id) {
  nvtxRangePushA(kKernelNames[id]);
  if (!h->prof) return;
  if (!h->ev[id][0]) {
    cudaEventCreate(&h->ev[id][0]);
    cudaEventCreate(&h->ev[id][1]);
  }
  cudaEventRecord(h->ev[id][0], h->stream);
}
void prof_end(pd_handle* h, int id) {
  nvtxRangePop();
  if (!h->prof) return;
  cudaEventRecord(h->ev[id][1], h->stream);
  h->ev_used[id] = true;
}
// after a stream sync: fold this iteration's event pairs into the accumulators
void prof_collect(pd_handle* h) {
  if (!h->prof) return;
  for (int i = 0; i < PD_NKERNELS; ++i)
    if (h->ev_used[i]) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, h->ev[i][0], h->ev[i][1]) == cudaSuccess) {
        h->prof_ms[i] += ms;
        h->prof_n[i] += 1;
      }
      h->ev_used[i] = false;
    }
}

template <typename T>
int dalloc(pd_handle* h, T** p, size_t count) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, count * sizeof(T) + 16);
  if (e != cudaSuccess)
    return fail(PD_ENOMEM, std::string("cudaMalloc(") + std::to_string(count * sizeof(T)) + "): " + cudaGetErrorString(e));
  h->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return PD_OK;
}

bool is_ch(int kind) { return kind == PD_CAHN_HILLIARD || kind == PD_CAHN_HILLIARD_EYRE; }
bool can_pipeline(const pd_handle* h);

int validate(const pd_problem* p) {
  if (!p) return fail(PD_EINVAL, "problem is NULL");
  if (p->kind < 0 || p->kind > 3) return fail(PD_EINVAL, "unknown kind");
  if (p->bc < 0 || p->bc > 1) return fail(PD_EINVAL, "unknown bc");
  if (p->dim != 1 && p->dim != 2) return fail(PD_EINVAL, "dim must be 1 or 2");
  if (is_ch(p->kind) && (p->dim != 2 || p->bc != PD_BC_NEUMANN))
    return fail(PD_EINVAL, "Cahn-Hilliard is supported in 2D with Neumann BCs (P:59)");
  {
    int n1, n2, ns1, ns2;
    int8_t pl1[12], pl2[12];
    const bool mixed = !is_pow2(p->nt) && mixed_split(p->nt, &n1, &n2, pl1, &ns1, pl2, &ns2);
    if (!((is_pow2(p->nt) && p->nt >= 2 && p->nt <= kMaxNt) || mixed))
      return fail(PD_EINVAL, "nt must be a power of two in [2, 2^20], or 2^a 5^b (>= 64) split as N1 N2 <= 1024^2 "
                             "(mixed-radix long-window path, e.g. 10^6 = 1000 x 1000, P:692)");
    if ((p->nt > kMaxNtShort || mixed) && p->dim == 1 && (!is_pow2(p->m) || p->m > 4096))
      return fail(PD_EINVAL, "1D long windows (nt > 4096 or mixed radix): m must be a power of two <= 4096");
  }
  if (p->dim == 2 && (!is_pow2(p->m) || p->m < 4 || p->m > 4096))
    return fail(PD_EINVAL, "2D: m (intervals per axis) must be a power of two in [4, 4096]");
  if (p->dim == 1 && (p->m < 4 || p->m > (1 << 20))) return fail(PD_EINVAL, "1D: m must be in [4, 2^20]");
  if (!(p->alpha > 0.0 && p->alpha < 1.0)) return fail(PD_EINVAL, "alpha must be in (0, 1) (P:308)");
  if (!(p->theta >= 0.5 && p->theta <= 1.0))
    return fail(PD_EINVAL, "theta must be in [1/2, 1] (theta-method, P:119-126; A-stable range)");
  if (is_ch(p->kind) && p->theta != 1.0)
    return fail(PD_EINVAL, "Cahn-Hilliard PinT-I is backward Euler (theta = 1, P:440-451)");
  if (!(p->t_window > 0.0) || !std::isfinite(p->t_window)) return fail(PD_EINVAL, "t_window must be > 0");
  if (!(p->eps >= 0.0)) return fail(PD_EINVAL, "eps must be >= 0");
  if (p->fixed_iters <= 0 && !(p->tol > 0.0)) return fail(PD_EINVAL, "tol must be > 0");
  if (p->n_windows < 1 || p->n_windows > PD_MAX_WINDOWS) return fail(PD_EINVAL, "n_windows out of range");
  if (p->fixed_iters <= 0 && p->max_iter < 1) return fail(PD_EINVAL, "max_iter must be >= 1");
  if (p->jacobian != PD_JACOBIAN_SCALAR && p->jacobian != PD_JACOBIAN_TIME_AVG)
    return fail(PD_EINVAL, "unknown jacobian");
  if (p->jacobian == PD_JACOBIAN_TIME_AVG && !is_ch(p->kind))
    return fail(PD_EINVAL, "the time-averaged Jacobian (P:486) is a Cahn-Hilliard option");
  if (is_ch(p->kind) && !(p->omega > 0.0 && p->tau > 0.0))
    return fail(PD_EINVAL, "CH damping needs omega > 0 and tau > 0");
  if (p->init != PD_INIT_BROADCAST && p->init != PD_INIT_ZERO) return fail(PD_EINVAL, "unknown init");
  return PD_OK;
}

void geometry(const pd_problem* p, int* nx, int* ny) {
  const int64_t n = p->bc == PD_BC_NEUMANN ? p->m + 1 : p->m - 1;
  *nx = (int)n;
  *ny = p->dim == 2 ? (int)n : 1;
}

double mu_of(const pd_problem* p, double Lam, double b2, double e2) {
  if (p->kind == PD_BIHARMONIC) return Lam * Lam;
  return b2 * Lam + e2 * (Lam * Lam);
}

template <typename K>
int allow_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) PD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return PD_OK;
}

size_t time_smem(int nt, int warps) { return (size_t)warps * padded16(nt) * sizeof(double2); }
size_t rows_smem(int M) { return (size_t)kLineWarps * dpadded(M) * sizeof(double); }
size_t cols_smem(int M, int w = kColW) { return ((size_t)w * dpadded(M) + 66 * w) * sizeof(double); }
// generic column pass: kColW columns per CTA, 4 when the line buffers would exceed shared memory (M = 4096)
int cols_per_cta(int M) { return cols_smem(M) <= kSmemMax ? kColW : 4; }

// ----------------------------------------------------------------------------- launches
int setup_fast_attrs(pd_handle* h) {
  if (!h->fast) return PD_OK;
  PD_CUDA(fast_attrs<1>());
  PD_CUDA(fast_attrs<2>());
  PD_CUDA(fast_attrs<4>());
  PD_CUDA(fast_attrs<8>());
  PD_CUDA(fast_attrs<16>());
  PD_CUDA(fast_attrs<32>());
  return PD_OK;
}

// k_x1d workspace row pitch: 2⌈N_x/2⌉ doubles (the time pass reads 16-byte pencil pairs)
// (N_x = 65: 80, so time slabs of 2, 4, 5 or 8 ranks get even column blocks; the pads stay zero)
size_t x1_pitch(const pd_handle* h) { return h->nx > 64 ? 80 : (size_t)((h->nx + 1) / 2) * 2; }

ResidualParams residual_params(pd_handle* h) {
  ResidualParams R;
  R.nx = h->nx; R.ny = h->ny; R.nt = h->P.nt; R.dim = h->P.dim;
  R.neumann = h->neumann; R.kind = h->P.kind;
  R.inv_h2 = h->inv_h2; R.inv_dt = h->inv_dt; R.b2 = h->b2; R.e2 = h->e2;
  R.y0g = 0; R.nyg = h->ny; R.hlo = nullptr; R.hhi = nullptr; R.theta = h->P.theta;
  R.dU = nullptr; R.unew = nullptr; R.umax = &h->st->umax_bits;
  R.ldr = h->nx; R.nsr = h->ns;
  return R;
}

// 1D long windows with N_x ≤ 64 (k_x1d.cuh): MODE 0 residual + forward x transform, 1 forward,
// 2 inverse (‖δ‖∞), 3 inverse + update
// nrows < 0: all N_t rows; bc > 0: the workspace side in time-slab column blocks of bc columns
// (block stride nrows·bc, X1Params)
int launch_x1d(pd_handle* h, int mode, const double* u0, const double* in, double* out, int kid,
               int64_t nrows = -1, int bc = 0) {
  X1Params Q;
  if (nrows < 0) nrows = h->P.nt;
  Q.nx = h->nx; Q.nt = (int)nrows; Q.R = residual_params(h); Q.B = h->x1T; Q.st = h->st;
  Q.ld_in = mode <= 1 ? h->nx : (int)x1_pitch(h);       // user arrays: N_x; workspace: even pitch
  Q.ld_out = mode <= 1 ? (int)x1_pitch(h) : h->nx;
  Q.bc = bc; Q.bstride = nrows * (int64_t)bc;
  const int units = (int)((nrows + 7) / 8);
  const unsigned grid = (unsigned)std::min((units + kX1Warps - 1) / kX1Warps, 148 * 2);
  prof_begin(h, kid);
  switch (mode) {
    case 0: k_x1d<0><<<grid, kX1Threads, kX1Smem, h->stream>>>(u0, in, out, Q); break;
    case 1: k_x1d<1><<<grid, kX1Threads, kX1Smem, h->stream>>>(u0, in, out, Q); break;
    case 2: k_x1d<2><<<grid, kX1Threads, kX1Smem, h->stream>>>(u0, in, out, Q); break;
    default: k_x1d<3><<<grid, kX1Threads, kX1Smem, h->stream>>>(u0, in, out, Q); break;
  }
  prof_end(h, kid);
  PD_LAUNCHED();
  return PD_OK;
}

// ldr != 0 (residual_to_wp): r is the padded workspace wp, row pitch ldr, slice pitch ny·ldr
int launch_residual(pd_handle* h, const double* u0, const double* U, double* r, const double* dU = nullptr,
                    double* unew = nullptr, int64_t ldr = 0) {
  ResidualParams R = residual_params(h);
  R.dU = dU; R.unew = unew;
  if (ldr) { R.ldr = ldr; R.nsr = (int64_t)h->ny * ldr; }
  const int kid = dU ? K_RESUPD : K_RESIDUAL;
  prof_begin(h, kid);
  size_t nparts = 0;     // CH: J̄ partial sums written by this launch (summed in a fixed order)
  if (h->P.dim == 2) {
    if ((h->tune & 32) && h->P.theta == 1.0 && h->P.kind != PD_CAHN_HILLIARD_EYRE) {     // previous row-streaming kernel (A/B)
      dim3 grd((h->nx + kResStrip - 1) / kResStrip, h->P.nt);
      k_residual_2d<<<grd, 128, 0, h->stream>>>(u0, U, r, R, h->jpart);
      nparts = (size_t)grd.x * grd.y;
    } else {
      dim3 grd((h->nx + kResTX - 1) / kResTX, (h->ny + kResTY - 1) / kResTY, (h->P.nt + kResChunk - 1) / kResChunk);
      if (dU && h->P.theta != 1.0)
        k_residual_tile<1, true><<<grd, kResThreads, kResSmemUpd, h->stream>>>(u0, U, r, R, h->jpart);
      else if (dU)
        k_residual_tile<0, true, 1><<<grd, kResThreads, kResSmemUpd, h->stream>>>(u0, U, r, R, h->jpart);
      else if (h->P.kind == PD_CAHN_HILLIARD_EYRE)
        k_residual_tile<2, false, 2><<<grd, kResThreads, kResSmem, h->stream>>>(u0, U, r, R, h->jpart);
      else if (h->P.theta != 1.0)
        k_residual_tile<1, false, 1><<<grd, kResThreads, kResSmem, h->stream>>>(u0, U, r, R, h->jpart);
      else if (!is_ch(h->P.kind) && ldr)
        k_residual_tile<0, false, 1, true><<<grd, kResThreads, kResSmem, h->stream>>>(u0, U, r, R, h->jpart);
      else if (!is_ch(h->P.kind))       // linear, single handle (launch_residual has no slab halos)
        k_residual_tile<0, false, 1><<<grd, kResThreads, kResSmem, h->stream>>>(u0, U, r, R, h->jpart);
      else                              // CH PinT-I, single handle
        k_residual_tile<0, false, 2><<<grd, kResThreads, kResSmem, h->stream>>>(u0, U, r, R, h->jpart);
      nparts = (size_t)grd.x * grd.y * grd.z;
    }
  } else {
    // 1D (linear kinds only): flattened grid-stride map
    int wlog = 5;
    while ((1 << wlog) < h->nx && wlog < 8) ++wlog;
    const int rpb = 256 >> wlog;
    const unsigned grid = (unsigned)std::min<int64_t>((h->P.nt + rpb - 1) / rpb, 148 * 16);
    k_residual_1d<<<grid, 256, 0, h->stream>>>(u0, U, r, R, wlog);
  }
  prof_end(h, kid);
  PD_LAUNCHED();
  if (is_ch(h->P.kind)) {
    prof_begin(h, K_JBAR);
    k_jbar_finalize<<<1, 1024, 0, h->stream>>>(h->jpart, nparts, 1.0 / (double)h->total, h->st);
    prof_end(h, K_JBAR);
    PD_LAUNCHED();
  }
  return PD_OK;
}

LineParams line_params(pd_handle* h, int axis, unsigned long long* amax, double* upd = nullptr) {
  LineParams L;
  L.nlines = (int64_t)h->P.nt * (axis == 0 ? h->ny : h->nx);
  L.nx = h->nx;
  L.ns = h->ns;
  L.ps_in = L.ps_out = L.ns;
  L.nel = h->nx;
  L.M = (int)h->P.m; L.log2h = h->log2h; L.trig = h->trig; L.tw = h->tw; L.twlog = h->twlog;
  L.trigs = h->trigsc; L.trigc = h->trigsc + std::max((int)h->P.m / 2, 1);
  L.amax = amax;
  L.tune = h->tune;
  L.upd = upd;
  L.oscale = nullptr;
  L.stagger_ns = h->stagger_ns;
  L.umax = upd ? &h->st->umax_bits : nullptr;
  L.sin.n = 0;
  L.sout.n = 0;
  L.ps_in = L.ps_out = h->ns;
  L.ldi = L.ldo = L.ldn = h->nx;
  return L;
}

FastLaunch fast_launch(pd_handle* h) {
  FastLaunch F;
  F.stream = h->stream; F.nt = h->P.nt; F.nx = h->nx; F.ns = h->ns; F.trig2 = h->trig2; F.dtt_ver = h->dtt_ver;
  F.trig2p = h->trig2p;
  return F;
}

bool fast_line_any(pd_handle* h, const double* in, double* out, int axis, const LineParams& L) {
  const FastLaunch F = fast_launch(h);
  const int nm = h->neumann ? 1 : 0;
  switch (L.M) {
    case 64: fast_line<1>(nm, axis, in, out, L, F); return true;
    case 128: fast_line<2>(nm, axis, in, out, L, F); return true;
    case 256: fast_line<4>(nm, axis, in, out, L, F); return true;
    case 512: fast_line<8>(nm, axis, in, out, L, F); return true;
    case 1024: fast_line<16>(nm, axis, in, out, L, F); return true;
    case 2048: fast_line<32>(nm, axis, in, out, L, F); return true;
    default: return false;
  }
}

int launch_lines(pd_handle* h, const double* in, double* out, int axis, unsigned long long* amax, int kid,
                 double* upd = nullptr, const double* oscale = nullptr, int64_t ps_in = 0, int64_t ps_out = 0,
                 int64_t ldi = 0, int64_t ldo = 0) {
  LineParams L = line_params(h, axis, amax, upd);
  L.oscale = oscale;
  if (ps_in) L.ps_in = ps_in;
  if (ps_out) L.ps_out = ps_out;
  if (ldi) L.ldi = ldi;                 // row passes: padded row pitch of in / out (wp)
  if (ldo) L.ldo = ldo;
  prof_begin(h, kid);
  const bool fast = h->fast && fast_line_any(h, in, out, axis, L);
  if (!fast) {
    if (axis == 0) {
      const unsigned grid = (unsigned)((L.nlines + kLineWarps - 1) / kLineWarps);
      const size_t smem = rows_smem(L.M);
      if (h->neumann) k_dtt_rows<1, kLineWarps><<<grid, kLineWarps * 32, smem, h->stream>>>(in, out, L);
      else k_dtt_rows<0, kLineWarps><<<grid, kLineWarps * 32, smem, h->stream>>>(in, out, L);
    } else {
      const int cw = cols_per_cta(L.M);
      const int64_t groups = (int64_t)h->P.nt * ((h->nx + cw - 1) / cw);
      const unsigned grid = (unsigned)std::min<int64_t>(groups, 148 * 64);
      const size_t smem = cols_smem(L.M, cw);
      if (cw == kColW) {
        if (h->neumann) k_dtt_cols<1, kColW><<<grid, kColW * 32, smem, h->stream>>>(in, out, L);
        else k_dtt_cols<0, kColW><<<grid, kColW * 32, smem, h->stream>>>(in, out, L);
      } else {
        if (h->neumann) k_dtt_cols<1, 4><<<grid, 4 * 32, smem, h->stream>>>(in, out, L);
        else k_dtt_cols<0, 4><<<grid, 4 * 32, smem, h->stream>>>(in, out, L);
      }
    }
  }
  prof_end(h, kid);
  PD_LAUNCHED();
  return PD_OK;
}

// y pass between the natural layout and the column-major wt (k_cols_cm): dir 0 forward, 1 inverse
int launch_cols_cm(pd_handle* h, int dir, const double* in, double* out, int kid, const double* oscale,
                   int64_t ldn = 0) {
  LineParams L = line_params(h, 1, nullptr);
  L.oscale = oscale;
  if (ldn) {                            // natural side in the padded workspace wp
    L.ldn = ldn;
    (dir == 0 ? L.ps_in : L.ps_out) = (int64_t)h->ny * ldn;
  }
  const FastLaunch F = fast_launch(h);
  const int nm = h->neumann ? 1 : 0;
  prof_begin(h, kid);
  switch (L.M) {
    case 64: fast_cols_cm<1>(nm, dir, in, out, L, F, h->lp); break;
    case 128: fast_cols_cm<2>(nm, dir, in, out, L, F, h->lp); break;
    case 256: fast_cols_cm<4>(nm, dir, in, out, L, F, h->lp); break;
    case 512: fast_cols_cm<8>(nm, dir, in, out, L, F, h->lp); break;
    case 1024: fast_cols_cm<16>(nm, dir, in, out, L, F, h->lp); break;
    case 2048: fast_cols_cm<32>(nm, dir, in, out, L, F, h->lp); break;
    default: return fail(PD_EINVAL, "column-major y pass: unsupported line length");
  }
  prof_end(h, kid);
  PD_LAUNCHED();
  return PD_OK;
}

// y⁻¹ from the column-major wt into the padded workspace wp through TMA box stores (M = 2048)
int launch_cols_tma_inv(pd_handle* h, const double* in, int kid, const double* oscale) {
  LineParams L = line_params(h, 1, nullptr);
  L.oscale = oscale;
  L.ldn = h->lpx;
  L.ps_out = (int64_t)h->ny * h->lpx;
  const FastLaunch F = fast_launch(h);
  const int nm = h->neumann ? 1 : 0;
  prof_begin(h, kid);
  bool ok = false;
  switch (L.M) {
    case 512: ok = fast_cols_tma_inv<8>(nm, in, L, F, h->lp, &h->wp_map); break;
    case 1024: ok = fast_cols_tma_inv<16>(nm, in, L, F, h->lp, &h->wp_map); break;
    case 2048: ok = fast_cols_tma_inv<32>(nm, in, L, F, h->lp, &h->wp_map); break;
    default: break;
  }
  prof_end(h, kid);
  if (!ok) return fail(PD_EINVAL, "TMA y-inverse pass: M = 512, 1024 or 2048 only");
  PD_LAUNCHED();
  return PD_OK;
}

bool fast_time_any(pd_handle* h, const double* in, double* out, const TimeParams& T) {
  if (!h->fast) return false;
  const FastLaunch F = fast_launch(h);
  switch (h->P.nt) {
    case 32: fast_time<1>(in, out, T, F); return true;
    case 64: fast_time<2>(in, out, T, F); return true;
    case 128: fast_time<4>(in, out, T, F); return true;
    case 256: fast_time<8>(in, out, T, F); return true;
    case 512: fast_time<16>(in, out, T, F); return true;
    case 1024: fast_time<32>(in, out, T, F); return true;
    default: return false;
  }
}

TimeParams time_params(pd_handle* h, unsigned long long* amax) {
  TimeParams T;
  T.nt = h->P.nt; T.log2nt = h->log2nt; T.ns = h->ns; T.nx = h->nx;
  T.gam = h->gam; T.ginv = h->ginv; T.dl = h->dl; T.el = h->el; T.l3 = h->l3; T.lamx = h->lam;
  T.kind = h->P.kind; T.b2 = h->b2; T.e2 = h->e2; T.st = h->st;
  T.tw = h->tw; T.twlog = h->twlog; T.amax = amax; T.tune = h->tune; T.xoff = 0;
  T.gamma_folded = 0;
  T.stagger_ns = h->stagger_ns;
  return T;
}

// Long-window time pass (k_tlong.cuh) on spatially transformed data: in → Y → X (divided) → Y → out.
// bc > 0 (time slabs, 1D): `in`/`out` hold the bc x-modes [c0, c0 + bc) of every time row (row
// pitch bc); the divide takes their eigenvalues through T.xoff.
int tlong_time(pd_handle* h, const double* in, double* out, int64_t c0 = 0, int64_t bc = 0) {
  TlongParams Q;
  Q.N = h->P.nt; Q.log2N = h->log2nt;
  Q.log2N1 = h->log2n1; Q.log2N2 = h->log2n2; Q.N1 = h->n1; Q.N2 = h->n2;
  Q.mixed = h->mixed ? 1 : 0;
  Q.mxp = h->mxp;
  Q.nst1 = h->nst1; Q.nst2 = h->nst2;
  for (int i = 0; i < 12; ++i) { Q.plan1[i] = h->plan1[i]; Q.plan2[i] = h->plan2[i]; }
  Q.mt1 = h->mtab; Q.mt2 = h->mtab ? h->mtab + h->n1 : nullptr; Q.mtN = h->mtab ? h->mtab + h->n1 + h->n2 : nullptr;
  Q.rev1 = h->mrev; Q.irev1 = h->mrev ? h->mrev + h->n1 : nullptr;
  Q.rev2 = h->mrev ? h->mrev + 2 * h->n1 : nullptr; Q.irev2 = h->mrev ? h->mrev + 2 * h->n1 + h->n2 : nullptr;
  Q.ns = h->ns; Q.P = (h->ns + 1) / 2; Q.nch = (Q.P + kTlPairs - 1) / kTlPairs;
  Q.ld = h->x1 ? (int64_t)x1_pitch(h) : h->ns;
  Q.ghi = h->tlg; Q.glo = h->tlg + Q.N1; Q.gihi = h->tlg + Q.N1 + Q.N2; Q.gilo = h->tlg + 2 * Q.N1 + Q.N2;
  Q.tw = h->tw; Q.twlog = h->twlog;
  Q.T = time_params(h, nullptr);
  if (bc > 0) {
    const int64_t ncol = std::min<int64_t>(bc, h->ns - c0);        // real modes in the block (pad excluded)
    Q.ns = ncol; Q.P = (ncol + 1) / 2; Q.nch = (Q.P + kTlPairs - 1) / kTlPairs; Q.ld = bc;
    Q.T.ns = ncol; Q.T.nx = (int)ncol; Q.T.xoff = (int)c0;
  }
  double2* Y = h->spec;
  double2* X = h->w1;
  if (h->tlfuse && tlong_fusable(Q)) {                   // A, fused B (+ divide), A⁻¹
    const int kid[3] = {K_TLA, K_TLBF, K_TLAI};
    const int stg[3] = {0, 5, 4};
    const void* ins[3] = {in, nullptr, Y};
    void* outs[3] = {Y, Y, out};
    for (int i = 0; i < 3; ++i) {
      prof_begin(h, kid[i]);
      if (!tlong_launch(stg[i], ins[i], outs[i], Q, h->stream)) return fail(PD_EINVAL, "tlong: unsupported N_t split");
      prof_end(h, kid[i]);
      PD_LAUNCHED();
    }
    return PD_OK;
  }
  const int kid[5] = {K_TLA, K_TLB, K_TLD, K_TLBI, K_TLAI};
  const void* ins[5] = {in, Y, nullptr, X, Y};
  void* outs[5] = {Y, X, X, Y, out};
  for (int stage = 0; stage < 5; ++stage) {
    prof_begin(h, kid[stage]);
    if (!tlong_launch(stage, ins[stage], outs[stage], Q, h->stream)) return fail(PD_EINVAL, "tlong: unsupported N_t split");
    prof_end(h, kid[stage]);
    PD_LAUNCHED();
  }
  return PD_OK;
}

// The last 2D pass (x-inverse, rows) can apply the update U += δ itself (k_rows3 epilogue): only
// the register-FFT v3 line kernels implement it.
bool can_fuse_update(const pd_handle* h) {
  // measured (d3f/d3g): the epilogue's U loads are exposed in the latency-bound line kernel, so the
  // fused pass (20.4 ms) loses to x-inverse + streaming update (10.3 + 8.2 ms) — opt-in (tune 16)
  return (h->tune & 16) && h->P.dim == 2 && !is_ch(h->P.kind) && h->fast && h->dtt_ver == 3 && h->P.m >= 64 &&
         h->P.m <= 2048;
}

// (A/B, opt-in: tune 2^26) 2D linear kinds with Neumann lines on the padded-workspace path (c5): the
// residual writes r into wp at its 64-byte aligned row pitch, so the forward x pass takes its rows
// by bulk copy like the inverse one (k_rows3 BK = 1) and runs in place.  Bit-identical; measured on
// c5: x 8.92 -> 8.49 ms but the residual 7.54 -> 8.33 ms (reading U at pitch 2049 while writing r
// at pitch 2056, with either form of the store addressing), 64.3 -> 64.7 ms per iteration: off.
bool residual_to_wp(pd_handle* h) {
  return h->P.dim == 2 && !is_ch(h->P.kind) && h->P.theta == 1.0 && h->neumann && h->P.m == 2048 && h->wt && h->wp &&
         h->dtt_ver == 3 && h->fast && !h->tlong && (h->tune & (1 << 26)) && !(h->tune & (65536 | 16 | 32)) &&
         h->P.jacobian != PD_JACOBIAN_TIME_AVG;
}

// δ = P_α⁻¹ r; with U_fused != NULL (can_fuse_update) the last pass adds δ to U_fused instead of
// storing δ (‖δ‖∞ and ‖U‖∞ reduced on the way).
// want_dmax = false: the caller's update folds ‖δ‖∞ (2D: the last x pass runs its plain variant).
// r_in_wp: r already lies in wp at its padded pitch (residual_to_wp), the forward x pass runs in place.
int precond(pd_handle* h, const double* r, double* delta, double* U_fused = nullptr, bool want_dmax = true,
            bool r_in_wp = false) {
  unsigned long long* dmax = &h->st->dmax_bits;
  if (h->P.dim == 2) {
    int rc;
    // when both the v3 column kernel and the register-FFT time pass run, the y passes carry
    // Γ_α (forward outputs) and Γ_α⁻¹·1/(N_t (2m)²) (inverse outputs) for the time pass
    const bool fold = !h->tlong && h->fast && h->dtt_ver >= 3 && h->P.m >= 64 && h->P.m <= 2048 && h->P.nt >= 32 &&
                      h->P.nt <= 1024;
    const bool use_wt = h->wt && h->dtt_ver == 3 && !(h->tune & 65536);   // tune 65536 (A/B): the in-place v2 time pass
    const bool use_wp = use_wt && h->wp;          // x, y passes exchange data through wp
    double* xo = use_wp ? h->wp : delta;           // x-pass output / x⁻¹-pass input
    if (r_in_wp && !use_wp) return fail(PD_EINVAL, "residual in wp without the padded-workspace path");
    if ((rc = launch_lines(h, r_in_wp ? h->wp : r, xo, 0, nullptr, K_XFWD, nullptr, nullptr, 0, 0, r_in_wp ? h->lpx : 0,
                           use_wp ? h->lpx : 0)))
      return rc;
    // (measured and not kept: TMA loads of the natural side through a 4-chunk staging ring, whole
    // tile 13.9 ms or half of it prefetched during the transform 14.4 ms, and TMA box stores of the
    // wt lines through the same ring 16.1 ms, against 12.3 ms for per-element cp.async + coalesced
    // register stores — the 64 KB ring takes the L1 that the transform's tables and the 8-byte
    // cp.async.ca column tile share; the inverse pass loads its wt lines by bulk copy, bypassing L1)
    if (use_wt) {
      if ((rc = launch_cols_cm(h, 0, xo, h->wt, K_YFWD, fold ? h->gam : nullptr, use_wp ? h->lpx : 0))) return rc;
    } else if ((rc = launch_lines(h, delta, delta, 1, nullptr, K_YFWD, nullptr, fold ? h->gam : nullptr))) {
      return rc;
    }
    TimeParams T = time_params(h, nullptr);
    T.gamma_folded = fold ? 1 : 0;
    bool done = false;
    if (use_wt) {                                 // TMA-staged three-stage time pass (k_time2d_v4)
      T.nx = (int)h->lp;                          // column-major wt: mode s = x·lp + y (Λ symmetric)
      T.ns = h->ps;
      CUtensorMap m;
      const unsigned rb = (unsigned)std::min<int64_t>(h->P.nt, 256);
      if (!make_map_2d(&m, h->wt, h->ps, h->P.nt, h->ps, 16, rb)) return fail(PD_ECUDA, "tensor map encode failed");
      // (T.nx, T.ns) = (lp, ps): every point of the padded column-major slice is a tile point
      const FastLaunch F = fast_launch(h);
      prof_begin(h, K_TIME);
      switch (h->P.nt) {
        case 32: done = fast_time_tma<1>(h->wt, T, F, &m); break;
        case 64: done = fast_time_tma<2>(h->wt, T, F, &m); break;
        case 128: done = fast_time_tma<4>(h->wt, T, F, &m); break;
        case 256: done = fast_time_tma<8>(h->wt, T, F, &m); break;
        case 512: done = fast_time_tma<16>(h->wt, T, F, &m); break;
        default: break;
      }
      prof_end(h, K_TIME);
      PD_LAUNCHED();
      if (!done) return fail(PD_EINVAL, "TMA time pass: unsupported N_t");
    }
    if (done) {
    } else if (h->tlong) {
      if ((rc = tlong_time(h, delta, delta))) return rc;
    } else {
    prof_begin(h, K_TIME);
    if (!fast_time_any(h, delta, delta, T)) {
      // generic time pass (N_t outside the register-FFT sizes): one pencil pair per warp, fewer
      // warps per CTA when the pencils are long (N_t = 2048/4096 need 35/70 KB per warp)
      if (time_smem(h->P.nt, kTimeWarps) <= kSmemMax) {
        const unsigned grid = (unsigned)((h->ns + 2 * kTimeWarps - 1) / (2 * kTimeWarps));
        k_time_solve_2d<kTimeWarps><<<grid, kTimeWarps * 32, time_smem(h->P.nt, kTimeWarps), h->stream>>>(delta, delta, T);
      } else {
        const unsigned grid = (unsigned)((h->ns + 1) / 2);
        k_time_solve_2d<1><<<grid, 32, time_smem(h->P.nt, 1), h->stream>>>(delta, delta, T);
      }
    }
    prof_end(h, K_TIME);
    PD_LAUNCHED();
    }
    if (use_wp) {
      if ((rc = launch_cols_tma_inv(h, h->wt, K_YINV, fold ? h->ginv : nullptr))) return rc;
    } else if (use_wt) {
      if ((rc = launch_cols_cm(h, 1, h->wt, delta, K_YINV, fold ? h->ginv : nullptr))) return rc;
    } else if ((rc = launch_lines(h, delta, delta, 1, nullptr, K_YINV, nullptr, fold ? h->ginv : nullptr))) {
      return rc;
    }
    const int64_t li = use_wp ? h->lpx : 0;
    if (U_fused) return launch_lines(h, xo, delta, 0, dmax, K_XINVUPD, U_fused, nullptr, 0, 0, li, 0);
    if ((rc = launch_lines(h, xo, delta, 0, want_dmax ? dmax : nullptr, K_XINV, nullptr, nullptr, 0, 0, li, 0))) return rc;
    return PD_OK;
  }
  if (h->tlong) {     // 1D long window: DST-I/DCT-I along x, four-step time pass with divide, inverse
    int rc;
    if (h->x1) {       // r̂, δ̂ in the workspace (even row pitch), r and δ in the caller's layout
      if ((rc = launch_x1d(h, 1, nullptr, r, h->work, K_XFWD))) return rc;
      if ((rc = tlong_time(h, h->work, h->work))) return rc;
      return launch_x1d(h, 2, nullptr, h->work, delta, K_XINV);
    }
    if ((rc = launch_lines(h, r, delta, 0, nullptr, K_XFWD))) return rc;
    if ((rc = tlong_time(h, delta, delta))) return rc;
    return launch_lines(h, delta, delta, 0, dmax, K_XINV);
  }
  TimeParams T = time_params(h, nullptr);
  const bool w4 = time_smem(h->P.nt, kTime1DWarps) <= kSmemMax;     // else one warp per CTA (N_t = 4096)
  const int nw = w4 ? kTime1DWarps : 1;
  const unsigned grid = (unsigned)((h->ns + 2 * nw - 1) / (2 * nw));
  const size_t smem = time_smem(h->P.nt, nw);
  prof_begin(h, K_TFWD1D);
  if (w4) k_time_fwd_1d<kTime1DWarps><<<grid, kTime1DWarps * 32, smem, h->stream>>>(r, h->spec, T);
  else k_time_fwd_1d<1><<<grid, 32, smem, h->stream>>>(r, h->spec, T);
  prof_end(h, K_TFWD1D);
  PD_LAUNCHED();
  PentaParams PP;
  PP.n = h->nx; PP.nb = h->nb; PP.neumann = h->neumann; PP.kind = h->P.kind;
  PP.inv_h2 = h->inv_h2; PP.b2 = h->b2; PP.e2 = h->e2; PP.band = h->band; PP.dl = h->dl; PP.el = h->el;
  const size_t nf = (size_t)h->nx * h->nb;
  PP.l1 = h->fac; PP.l2 = h->fac + nf; PP.iu0 = h->fac + 2 * nf; PP.u1 = h->fac + 3 * nf;
  PP.refine = h->penta_refine;
  prof_begin(h, K_PENTA);
  if (h->nx <= kPentaCtaMaxN && h->penta_cta)        // one CTA per bin, everything in shared memory
    k_penta_solve_cta<<<h->nb, kPentaCtaThreads, penta_cta_smem(h->nx), h->stream>>>(h->spec, PP);
  else
    k_penta_solve<<<(h->nb + 63) / 64, 64, 0, h->stream>>>(h->spec, h->w1, h->w2, PP);
  prof_end(h, K_PENTA);
  PD_LAUNCHED();
  T.amax = dmax;
  prof_begin(h, K_TINV1D);
  if (w4) k_time_inv_1d<kTime1DWarps><<<grid, kTime1DWarps * 32, smem, h->stream>>>(h->spec, delta, T);
  else k_time_inv_1d<1><<<grid, 32, smem, h->stream>>>(h->spec, delta, T);
  prof_end(h, K_TINV1D);
  PD_LAUNCHED();
  return PD_OK;
}

// ---- NEXT-4: Step-(2) with the time-averaged Jacobian (k_krylov.cuh) -------------------------
constexpr int kKryM = kKryMaxM;      // GMRES restart length
constexpr int kKryCycles = 20;       // restarts before PD_NOT_CONVERGED
constexpr double kKryTol = 1e-13;    // relative preconditioned residual

unsigned kgrid(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8); }

// dots of V_0..V_{nv-1} (stride total) with y → h->khost[0..nv) (synchronises; folds profiled events)
int kdots(pd_handle* h, const double* V, int nv, const double* y) {
  prof_begin(h, K_KVEC);
  k_mdot<<<kKryBlocks, kKryThreads, 0, h->stream>>>(V, h->total, nv, y, h->total, h->kpart);
  k_mdot_final<<<nv, 256, 0, h->stream>>>(h->kpart, kKryBlocks, h->kdev);
  prof_end(h, K_KVEC);
  PD_LAUNCHED();
  PD_CUDA(cudaMemcpyAsync(h->khost, h->kdev, nv * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  PD_CUDA(cudaStreamSynchronize(h->stream));
  prof_collect(h);
  return PD_OK;
}

// y += s · Σ_{i<nv} c_i V_i with c = h->khost[0..nv) (uploaded)
int kcombine(pd_handle* h, double* y, const double* V, int nv, double s) {
  PD_CUDA(cudaMemcpyAsync(h->kdev, h->khost, nv * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  prof_begin(h, K_KVEC);
  k_maxpy<<<kgrid(h->total), 256, 0, h->stream>>>(y, V, h->total, nv, h->kdev, s, h->total);
  prof_end(h, K_KVEC);
  PD_LAUNCHED();
  return PD_OK;
}

int kaxpby(pd_handle* h, double* y, const double* x, double a, double b) {
  k_axpby<<<kgrid(h->total), 256, 0, h->stream>>>(y, x, a, b, h->total);
  PD_LAUNCHED();
  return PD_OK;
}

// w' = jt - c - J̄ and J̄ = mean(jt) - c into the device stats (c = 1 PinT-I, 0 PinT-II)
int setup_wprime(pd_handle* h, const double* jt) {
  const double c = h->P.kind == PD_CAHN_HILLIARD ? 1.0 : 0.0;
  k_block_sum<<<kKryBlocks, kKryThreads, 0, h->stream>>>(jt, h->ns, h->kpart);
  k_wprime<<<kgrid(h->ns), 256, 0, h->stream>>>(jt, h->kpart, kKryBlocks, h->ns, c, h->wfld, h->st);
  PD_LAUNCHED();
  return PD_OK;
}

// out = K x = P(J̄)⁻¹ Δ_h(w' ⊙ x)   (out may not alias x)
int apply_K(pd_handle* h, const double* x, double* out) {
  prof_begin(h, K_KLAP);
  k_lap_w<<<kgrid(h->total), 256, 0, h->stream>>>(x, h->wfld, out, h->nx, h->ny, h->P.nt, h->inv_h2);
  prof_end(h, K_KLAP);
  PD_LAUNCHED();
  return precond(h, out, out);
}

// One cycle's Arnoldi steps as a conditional WHILE graph (k_krylov.cuh, device-side Arnoldi): the
// body applies K to V_j through the fixed vectors kin / kout, orthogonalises (cgs_passes classical
// Gram-Schmidt passes), normalises and lets k_kry_tail update the Givens QR and decide.  Built once
// per handle (every pointer it uses is the handle's).
int build_kry_graph(pd_handle* h) {
  if (!h->kin) {
    int rc;
    if ((rc = dalloc(h, &h->kin, (size_t)h->total)) || (rc = dalloc(h, &h->kout, (size_t)h->total)) ||
        (rc = dalloc(h, &h->kd, 1)))
      return rc;
    PD_CUDA(cudaMallocHost(&h->kd_host, sizeof(KryDev)));
  }
  if (!h->cap_stream) PD_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
  PD_CUDA(cudaGraphCreate(&h->kgraph, 0));
  PD_CUDA(cudaGraphConditionalHandleCreate(&h->kcond, h->kgraph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h->kcond;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  PD_CUDA(cudaGraphAddNode(&node, h->kgraph, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  cudaStream_t saved = h->stream;
  h->stream = h->cap_stream;
  int rc = PD_OK;
  const int64_t n = h->total;
  const unsigned g = kgrid(n);
  if (cudaStreamBeginCaptureToGraph(h->cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
      cudaSuccess) {
    rc = fail(PD_ECUDA, "Krylov graph capture begin");
  } else {
    cudaStream_t st = h->cap_stream;
    k_kry_copy_in<<<g, 256, 0, st>>>(h->kV, n, h->kd, h->kin);
    PD_LAUNCHED();
    k_lap_w<<<g, 256, 0, st>>>(h->kin, h->wfld, h->kout, h->nx, h->ny, h->P.nt, h->inv_h2);
    PD_LAUNCHED();
    rc = precond(h, h->kout, h->kout);                                  // K v_j
    if (rc == PD_OK) {
      k_kry_sub<<<g, 256, 0, st>>>(h->kV, n, h->kd, h->kin, h->kout);   // A v_j = v_j - K v_j
      for (int pass = 0; pass < h->cgs_passes; ++pass) {
        k_kry_mdot<false><<<kKryBlocks, kKryThreads, 0, st>>>(h->kV, n, h->kd, h->kpart);
        k_kry_final<false><<<kKryM + 1, 256, 0, st>>>(h->kpart, kKryBlocks, h->kd);
        k_kry_maxpy<<<g, 256, 0, st>>>(h->kV, n, h->kd);
      }
      k_kry_mdot<true><<<kKryBlocks, kKryThreads, 0, st>>>(h->kV, n, h->kd, h->kpart);
      k_kry_final<true><<<1, 256, 0, st>>>(h->kpart, kKryBlocks, h->kd);
      k_kry_tail<<<1, 1, 0, st>>>(h->kd, h->kcond);
      k_kry_scale<<<g, 256, 0, st>>>(h->kV, n, h->kd);
      PD_LAUNCHED();
    }
    cudaGraph_t captured = nullptr;
    const cudaError_t e = cudaStreamEndCapture(h->cap_stream, &captured);
    if (rc == PD_OK && e != cudaSuccess) rc = fail(PD_ECUDA, std::string("Krylov graph capture: ") + cudaGetErrorString(e));
  }
  h->stream = saved;
  if (rc) return rc;
  PD_CUDA(cudaGraphInstantiate(&h->kgexec, h->kgraph, 0));
  return PD_OK;
}

// δ = G̃'⁻¹ r: GMRES(kKryM) on (I - K) δ = P⁻¹ r, started from δ₀ = P⁻¹ r (the scalar-J̄ solution),
// classical Gram-Schmidt applied twice, Givens rotations on the host.  r and delta may alias.
int precond_jt(pd_handle* h, const double* r, double* delta) {
  const int64_t n = h->total;
  double* V = h->kV;
  double* b = h->kb;
  int rc;
  const bool use_graph = h->kry_graph && !h->prof;                    // events cannot be captured
  if (use_graph && !h->kgexec && (rc = build_kry_graph(h))) return rc;
  if ((rc = precond(h, r, delta))) return rc;                         // δ₀ = b' = P⁻¹ r
  PD_CUDA(cudaMemcpyAsync(b, delta, n * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  if ((rc = kdots(h, b, 1, b))) return rc;
  const double bn = std::sqrt(h->khost[0]);
  std::vector<double> H((size_t)(kKryM + 1) * kKryM, 0.0), cs(kKryM), sn(kKryM), g(kKryM + 1), y(kKryM);
  auto Hij = [&](int i, int j) -> double& { return H[(size_t)i * kKryM + j]; };
  bool conv = bn == 0.0;
  int steps = 0;
  // each cycle starts from the TRUE preconditioned residual, so convergence is only declared on it
  for (int cyc = 0; cyc <= kKryCycles && !conv; ++cyc) {
    // b' - (δ - Kδ) into V_0
    if ((rc = apply_K(h, delta, V))) return rc;                       // V_0 = Kδ
    if ((rc = kaxpby(h, V, delta, -1.0, 1.0))) return rc;             // Kδ - δ
    if ((rc = kaxpby(h, V, b, 1.0, 1.0))) return rc;                  // + b'
    if ((rc = kdots(h, V, 1, V))) return rc;
    const double beta = std::sqrt(h->khost[0]);
    if (!std::isfinite(beta)) return fail(PD_EDIVERGED, "inner GMRES: non-finite residual");
    if (beta <= kKryTol * bn) {
      conv = true;
      break;
    }
    if (cyc == kKryCycles) break;
    if ((rc = kaxpby(h, V, V, 1.0 / beta - 1.0, 1.0))) return rc;    // V_0 /= β
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int j = 0;
    if (use_graph) {                                                  // the cycle's steps on the device
      KryDev* k = h->kd_host;
      std::memset(k, 0, sizeof(KryDev));
      k->bn = bn;
      k->tol = kKryTol;
      k->g[0] = beta;
      PD_CUDA(cudaMemcpyAsync(h->kd, k, sizeof(KryDev), cudaMemcpyHostToDevice, h->stream));
      PD_CUDA(cudaGraphLaunch(h->kgexec, h->stream));
      PD_CUDA(cudaMemcpyAsync(k, h->kd, sizeof(KryDev), cudaMemcpyDeviceToHost, h->stream));
      PD_CUDA(cudaStreamSynchronize(h->stream));
      j = k->j;
      steps += k->steps;
      for (int i = 0; i <= kKryM; ++i) g[i] = k->g[i];
      for (int i = 0; i < (kKryM + 1) * kKryM; ++i) H[i] = k->H[i];
    }
    for (; !use_graph && j < kKryM; ++j) {
      double* vj = V + (size_t)j * n;
      double* vn = V + (size_t)(j + 1) * n;
      if ((rc = apply_K(h, vj, vn))) return rc;                       // K v_j
      if ((rc = kaxpby(h, vn, vj, 1.0, -1.0))) return rc;             // A v_j = v_j - K v_j
      for (int pass = 0; pass < h->cgs_passes; ++pass) {              // classical Gram-Schmidt
        if ((rc = kdots(h, V, j + 1, vn))) return rc;
        for (int i = 0; i <= j; ++i) Hij(i, j) += h->khost[i];
        if ((rc = kcombine(h, vn, V, j + 1, -1.0))) return rc;
      }
      if ((rc = kdots(h, vn, 1, vn))) return rc;
      const double hn = std::sqrt(h->khost[0]);
      Hij(j + 1, j) = hn;
      if (hn > 0.0 && (rc = kaxpby(h, vn, vn, 1.0 / hn - 1.0, 1.0))) return rc;
      for (int i = 0; i < j; ++i) {                                   // previous rotations
        const double a = Hij(i, j), c2 = Hij(i + 1, j);
        Hij(i, j) = cs[i] * a + sn[i] * c2;
        Hij(i + 1, j) = -sn[i] * a + cs[i] * c2;
      }
      const double a = Hij(j, j), c2 = Hij(j + 1, j), rr = std::hypot(a, c2);
      cs[j] = rr > 0.0 ? a / rr : 1.0;
      sn[j] = rr > 0.0 ? c2 / rr : 0.0;
      Hij(j, j) = rr;
      Hij(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++steps;
      if (std::fabs(g[j + 1]) <= kKryTol * bn || hn == 0.0) {
        ++j;
        break;
      }
    }
    if (j > kKryM) j = kKryM;
    for (int i = j - 1; i >= 0; --i) {                                // back substitution
      double t = g[i];
      for (int k = i + 1; k < j; ++k) t -= Hij(i, k) * y[k];
      y[i] = t / Hij(i, i);
    }
    for (int i = 0; i < j; ++i) h->khost[i] = y[i];
    if ((rc = kcombine(h, delta, V, j, 1.0))) return rc;
    std::fill(H.begin(), H.end(), 0.0);
  }
  h->kry_last = steps;
  k_reset_dmax<<<1, 1, 0, h->stream>>>(h->st);
  k_amax_stats<<<kgrid(n), 256, 0, h->stream>>>(delta, n, h->st);
  PD_LAUNCHED();
  return conv ? PD_OK : PD_NOT_CONVERGED;
}

int launch_update(pd_handle* h, double* U, const double* delta, bool want_dmax = false) {
  const int damped = is_ch(h->P.kind);
  prof_begin(h, K_UPDATE);
  k_update<<<148 * 8, 256, 0, h->stream>>>(U, delta, (size_t)h->total, h->st, damped, h->P.omega, h->P.tau, nullptr,
                                            want_dmax && !damped ? 1 : 0);
  prof_end(h, K_UPDATE);
  PD_LAUNCHED();
  return PD_OK;
}

int init_iterate(pd_handle* h, double* U, const double* u0) {
  k_init_iterate<<<148 * 8, 256, 0, h->stream>>>(U, u0, (size_t)h->ns, (size_t)h->total,
                                                  h->P.init == PD_INIT_ZERO);
  PD_LAUNCHED();
  return PD_OK;
}

// One iteration's kernels (no host synchronisation except inside the NEXT-4 inner solve).
int enqueue_iteration(pd_handle* h, const double* u0, double* U) {
  int rc;
  k_reset_stats<<<1, 1, 0, h->stream>>>(h->st);
  PD_LAUNCHED();
  if (h->P.jacobian == PD_JACOBIAN_TIME_AVG) {   // NEXT-4: J̃ = diag(mean_n 3U²), inner GMRES
    if ((rc = launch_residual(h, u0, U, h->work))) return rc;
    k_tavg_jt<<<kgrid(h->ns), 256, 0, h->stream>>>(U, h->jt, h->ns, h->P.nt);
    PD_LAUNCHED();
    if ((rc = setup_wprime(h, h->jt))) return rc;
    if ((rc = precond_jt(h, h->work, h->work)) < 0) return rc;  // PD_NOT_CONVERGED: inexact step, continue
    if ((rc = launch_update(h, U, h->work))) return rc;
  } else if (h->x1) {    // residual + x transform, time pass, x inverse + update: 7 passes
    if ((rc = launch_x1d(h, 0, u0, U, h->work, K_XRES))) return rc;
    if ((rc = tlong_time(h, h->work, h->work))) return rc;
    if ((rc = launch_x1d(h, 3, nullptr, h->work, U, K_XUPD))) return rc;
  } else if (residual_to_wp(h)) {   // r straight into wp: the forward x pass bulk-loads its rows, in place
    if ((rc = launch_residual(h, u0, U, h->wp, nullptr, nullptr, h->lpx))) return rc;
    if ((rc = precond(h, h->wp, h->work, nullptr, false, true))) return rc;
    if ((rc = launch_update(h, U, h->work, true))) return rc;
  } else if ((rc = launch_residual(h, u0, U, h->work))) {
    return rc;
  } else if (can_fuse_update(h)) {
    if ((rc = precond(h, h->work, h->work, U))) return rc;
  } else {
    // ω = 1 (linear kinds, 2D): ‖δ‖∞ rides in the HBM-bound update instead of the last line pass
    // (measured c5: x⁻¹ 10.08 → 9.5 ms); the damped CH step needs ‖δ‖∞ before the update
    const bool upd_dmax = !is_ch(h->P.kind) && h->P.dim == 2;
    if ((rc = precond(h, h->work, h->work, nullptr, !upd_dmax))) return rc;
    if ((rc = launch_update(h, U, h->work, upd_dmax))) return rc;
  }
  return PD_OK;
}

int iteration(pd_handle* h, const double* u0, double* U, pd_iter_info* info) {
  int rc;
  if ((rc = enqueue_iteration(h, u0, U))) return rc;
  PD_CUDA(cudaMemcpyAsync(h->st_host, h->st, sizeof(DevStats), cudaMemcpyDeviceToHost, h->stream));
  PD_CUDA(cudaStreamSynchronize(h->stream));
  prof_collect(h);
  double dmax, umax;
  std::memcpy(&dmax, &h->st_host->dmax_bits, sizeof(double));
  std::memcpy(&umax, &h->st_host->umax_bits, sizeof(double));
  info->delta_max = dmax;
  info->u_max = umax;
  info->rel = umax > 0 ? dmax / umax : 0.0;
  info->jbar = is_ch(h->P.kind) ? h->st_host->jbar : 0.0;
  info->omega = h->st_host->omega;
  if (!std::isfinite(dmax) || !std::isfinite(umax)) return fail(PD_EDIVERGED, "non-finite increment or iterate");
  return PD_OK;
}

// ---- device-side window loop (CUDA graph with a conditional WHILE node; SURVEY §8(a) a5 "scalars
// to host or graph conditional"): the body is one iteration's kernels plus k_loop_decide, which
// applies the stop rule on the device — no host round trip per iteration
struct LoopCtl {
  int iters, limit, fixed, status;   // status: 0 running, 1 converged, 2 iteration limit, 3 non-finite,
                                     // 4 diverging (PD_GROWTH_LIMIT consecutive growths of ‖δ‖∞)
  int growth, diverging;
  double tol, rel, dmax, umax;
};

__global__ void k_loop_decide(const DevStats* st, LoopCtl* c, cudaGraphConditionalHandle cond) {
  const double dmax = __longlong_as_double((long long)st->dmax_bits);
  const double umax = __longlong_as_double((long long)st->umax_bits);
  const int it = ++c->iters;
  const bool finite = isfinite(dmax) && isfinite(umax);
  const bool conv = c->fixed <= 0 && dmax <= c->tol * umax;           // R#4, as the host loop
  c->growth = (it > 1 && dmax > c->dmax) ? c->growth + 1 : 0;
  if (c->growth >= PD_GROWTH_LIMIT) c->diverging = 1;
  const bool stop_div = c->diverging && c->fixed <= 0 && !conv;
  c->status = !finite ? 3 : conv ? 1 : stop_div ? 4 : (it >= c->limit ? 2 : 0);
  c->rel = umax > 0 ? dmax / umax : 0.0;
  c->dmax = dmax;
  c->umax = umax;
  cudaGraphSetConditional(cond, c->status == 0 ? 1 : 0);
}

bool can_pipeline(const pd_handle* h);

bool graph_ok(const pd_handle* h) {
  return h->use_graph && !h->prof && !h->slab && h->P.jacobian == PD_JACOBIAN_SCALAR && !can_pipeline(h);
}

// Capture one iteration (reading u0 from the hand-off buffer, iterating on U) plus the stop rule
// as the body of a conditional WHILE node.  Captured on a private stream (the caller's may be the
// legacy default stream, which cannot be captured); launched on the caller's.
int build_graph(pd_handle* h, double* U) {
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->graph) cudaGraphDestroy(h->graph);
  h->gexec = nullptr;
  h->graph = nullptr;
  h->gU = nullptr;
  if (!h->cap_stream) PD_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
  if (!h->ctl) {
    LoopCtl* c = nullptr;
    int rc = dalloc(h, &c, 1);
    if (rc) return rc;
    h->ctl = c;
  }
  if (!h->ctl_host) PD_CUDA(cudaMallocHost(&h->ctl_host, sizeof(LoopCtl)));
  PD_CUDA(cudaGraphCreate(&h->graph, 0));
  PD_CUDA(cudaGraphConditionalHandleCreate(&h->gcond, h->graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h->gcond;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  PD_CUDA(cudaGraphAddNode(&node, h->graph, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  cudaStream_t saved = h->stream;
  h->stream = h->cap_stream;
  int rc = PD_OK;
  if (cudaStreamBeginCaptureToGraph(h->cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
      cudaSuccess) {
    rc = fail(PD_ECUDA, "graph capture begin");
  } else {
    rc = enqueue_iteration(h, h->u0buf, U);
    if (rc == PD_OK) k_loop_decide<<<1, 1, 0, h->cap_stream>>>(h->st, static_cast<LoopCtl*>(h->ctl), h->gcond);
    cudaGraph_t captured = nullptr;
    const cudaError_t e = cudaStreamEndCapture(h->cap_stream, &captured);
    if (rc == PD_OK && e != cudaSuccess) rc = fail(PD_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  }
  h->stream = saved;
  if (rc) return rc;
  PD_CUDA(cudaGraphInstantiate(&h->gexec, h->graph, 0));
  h->gU = U;
  return PD_OK;
}

// One window on the device: reset the loop control, launch the graph, read the outcome.
int graph_window(pd_handle* h, int* iters, bool* conv, double* rel, bool* div) {
  LoopCtl* c = static_cast<LoopCtl*>(h->ctl_host);
  *c = LoopCtl{};
  c->fixed = h->P.fixed_iters;
  c->limit = h->P.fixed_iters > 0 ? h->P.fixed_iters : h->P.max_iter;
  c->tol = h->P.tol;
  PD_CUDA(cudaMemcpyAsync(h->ctl, c, sizeof(LoopCtl), cudaMemcpyHostToDevice, h->stream));
  PD_CUDA(cudaGraphLaunch(h->gexec, h->stream));
  PD_CUDA(cudaMemcpyAsync(c, h->ctl, sizeof(LoopCtl), cudaMemcpyDeviceToHost, h->stream));
  PD_CUDA(cudaStreamSynchronize(h->stream));
  *iters = c->iters;
  *conv = c->status == 1;
  *rel = c->rel;
  *div = c->diverging != 0;
  if (c->status == 3) return fail(PD_EDIVERGED, "non-finite increment or iterate");
  return PD_OK;
}

bool can_pipeline(const pd_handle* h) {
  return h->pipe && !h->slab && h->P.dim == 2 && !is_ch(h->P.kind) && h->fast && h->P.m >= 64 && h->P.m <= 2048 &&
         h->P.nt >= 32 && h->P.nt <= 1024;
}

int read_stats(pd_handle* h, double* dmax, double* umax) {
  PD_CUDA(cudaMemcpyAsync(h->st_host, h->st, sizeof(DevStats), cudaMemcpyDeviceToHost, h->stream));
  PD_CUDA(cudaStreamSynchronize(h->stream));
  prof_collect(h);
  std::memcpy(dmax, &h->st_host->dmax_bits, sizeof(double));
  std::memcpy(umax, &h->st_host->umax_bits, sizeof(double));
  return PD_OK;
}

// One window of the pipelined solve (can_pipeline): the same iterates as the plain loop —
//   step 1:  r = b - K U⁰, δ_1 = P⁻¹ r
//   step k:  U^{k-1} = U^{k-2} + δ_{k-1} (inside the residual, written to the other U buffer),
//            r = b - K U^{k-1}, δ_k = P⁻¹ r
//   end:     U^K = U^{K-1} + δ_K into the caller's buffer
// which saves the separate update pass (24 B/dof).  The stop test of iteration k-1 (needs ‖U^{k-1}‖)
// runs after step k; on convergence step k's δ is discarded.
int solve_window_pipelined(pd_handle* h, const double* u0, double* U, int* iters, bool* conv, double* rel,
                           bool* div) {
  if (!h->Ub) {
    int rc;
    if ((rc = dalloc(h, &h->Ub, (size_t)h->total)) || (rc = dalloc(h, &h->work2, (size_t)h->total))) return rc;
  }
  double* Ubuf[2] = {U, h->Ub};
  double* Wbuf[2] = {h->work, h->work2};
  int cu = 0, cw = 0, rc;
  const bool fixed = h->P.fixed_iters > 0;
  const int kmax = fixed ? h->P.fixed_iters : h->P.max_iter;
  if ((rc = init_iterate(h, U, u0))) return rc;
  k_reset_stats<<<1, 1, 0, h->stream>>>(h->st);
  PD_LAUNCHED();
  if ((rc = launch_residual(h, u0, U, Wbuf[0]))) return rc;
  if ((rc = precond(h, Wbuf[0], Wbuf[0]))) return rc;
  double dmax = 0, umax = 0, dprev = 0;
  if ((rc = read_stats(h, &dprev, &umax))) return rc;
  if (!std::isfinite(dprev)) return fail(PD_EDIVERGED, "non-finite increment");
  *conv = false;
  *div = false;
  int growth = 0;
  for (int k = 2; k <= kmax; ++k) {
    k_reset_stats<<<1, 1, 0, h->stream>>>(h->st);
    PD_LAUNCHED();
    if ((rc = launch_residual(h, u0, Ubuf[cu], Wbuf[1 - cw], Wbuf[cw], Ubuf[1 - cu]))) return rc;
    cu = 1 - cu;
    cw = 1 - cw;
    if ((rc = precond(h, Wbuf[cw], Wbuf[cw]))) return rc;
    if ((rc = read_stats(h, &dmax, &umax))) return rc;          // ‖δ_k‖, ‖U^{k-1}‖
    if (!std::isfinite(dmax) || !std::isfinite(umax)) return fail(PD_EDIVERGED, "non-finite increment or iterate");
    if (!fixed && dprev <= h->P.tol * umax) {                   // iteration k-1 converged
      *conv = true;
      *iters = k - 1;
      *rel = umax > 0 ? dprev / umax : 0.0;
      if (Ubuf[cu] != U)
        PD_CUDA(cudaMemcpyAsync(U, Ubuf[cu], (size_t)h->total * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
      return PD_OK;
    }
    growth = dmax > dprev ? growth + 1 : 0;                      // SURVEY §5.3 (PD_GROWTH_LIMIT)
    dprev = dmax;
    if (growth >= PD_GROWTH_LIMIT) {
      *div = true;
      if (!fixed) {                                             // stop: U^k = U^{k-1} + δ_k below
        *iters = k;
        break;
      }
    }
  }
  if (*div && !fixed) {
    k_reset_stats<<<1, 1, 0, h->stream>>>(h->st);
    PD_LAUNCHED();
    k_update<<<148 * 8, 256, 0, h->stream>>>(U, Wbuf[cw], (size_t)h->total, h->st, 0, 1.0, 1.0, Ubuf[cu]);
    PD_LAUNCHED();
    if ((rc = read_stats(h, &dmax, &umax))) return rc;
    *rel = umax > 0 ? dprev / umax : 0.0;
    return PD_OK;
  }
  k_reset_stats<<<1, 1, 0, h->stream>>>(h->st);
  PD_LAUNCHED();
  prof_begin(h, K_UPDATE);
  k_update<<<148 * 8, 256, 0, h->stream>>>(U, Wbuf[cw], (size_t)h->total, h->st, 0, 1.0, 1.0, Ubuf[cu]);
  prof_end(h, K_UPDATE);
  PD_LAUNCHED();
  if ((rc = read_stats(h, &dmax, &umax))) return rc;
  if (!std::isfinite(umax)) return fail(PD_EDIVERGED, "non-finite iterate");
  *iters = kmax;
  *rel = umax > 0 ? dprev / umax : 0.0;
  *conv = !fixed && dprev <= h->P.tol * umax;
  return PD_OK;
}

int check_handle(pd_handle* h) {
  if (!h) return fail(PD_EINVAL, "handle is NULL");
  PD_CUDA(cudaSetDevice(h->device));
  return PD_OK;
}

}  // namespace

extern "C" {

int paradiag_abi_version(void) { return PARADIAG_ABI_VERSION; }

const char* paradiag_strerror(int code) {
  switch (code) {
    case PD_OK: return "PD_OK";
    case PD_NOT_CONVERGED: return "PD_NOT_CONVERGED";
    case PD_EINVAL: return "PD_EINVAL: invalid problem or argument";
    case PD_ESINGULAR: return "PD_ESINGULAR: singular shifted system";
    case PD_ECUDA: return "PD_ECUDA: CUDA failure";
    case PD_ENCCL: return "PD_ENCCL: communicator failure";
    case PD_ENOMEM: return "PD_ENOMEM: device allocation failed";
    case PD_EDIVERGED: return "PD_EDIVERGED: non-finite values";
    default: return "unknown paradiag status";
  }
}

const char* paradiag_last_error(void) { return g_last_error.c_str(); }

int paradiag_workspace_bytes(const pd_problem* p, int nranks, size_t* bytes) {
  int rc = validate(p);
  if (rc) return rc;
  if (!bytes) return fail(PD_EINVAL, "bytes is NULL");
  if (nranks > 1) {                  // per rank: row slab, column slab, transpose buffer, halos, tables
    int nx, ny;
    geometry(p, &nx, &ny);
    const size_t per = (size_t)p->nt * nx * ((ny + nranks - 1) / nranks);
    *bytes = (5 * per + 4 * (size_t)p->nt * 2 * nx) * sizeof(double) +
             (size_t)(1 << std::max(ilog2(p->nt), ilog2(p->m))) * sizeof(double2);
    return PD_OK;
  }
  int nx, ny;
  geometry(p, &nx, &ny);
  const size_t ns = (size_t)nx * ny, total = ns * p->nt, nb = p->nt / 2 + 1;
  size_t b = total * sizeof(double) + ns * sizeof(double);
  const bool tl = p->nt > kMaxNtShort || !is_pow2(p->nt);
  if (tl) b += 2 * (size_t)p->nt * ((ns + 1) / 2) * sizeof(double2);       // Y, X of k_tlong.cuh
  else if (p->dim == 1) b += 7 * (size_t)nx * nb * sizeof(double2) + 5 * (size_t)nx * sizeof(double);
  b += (size_t)p->nt * (2 * sizeof(double) + sizeof(double2)) + (size_t)(p->m + 2) * (sizeof(double) + sizeof(double2));
  b += (size_t)(1 << std::max(ilog2(p->nt), ilog2(p->m))) * sizeof(double2);
  // TMA time pass workspace (2D, 32 <= nt <= 512, 64 <= m <= 2048): one more iterate-sized array
  if (p->dim == 2 && !tl && p->nt >= 32 && p->nt <= 512 && p->m >= 64 && p->m <= 2048) {
    b += p->nt * (ns + 1) * sizeof(double);
    // M = 2048 (M = 512 / 1024 with PARADIAG_WP=1): the padded x/y exchange workspace wp (rows
    // rounded up to 8 doubles)
    if (p->m == 2048) b += (size_t)p->nt * ny * ((nx + 7) & ~7) * sizeof(double);
  }
  // (the opt-in pipelined solve, PARADIAG_PIPELINE=1, adds 2 more iterate-sized arrays)
  // NEXT-4: the GMRES basis (kKryM + 1), b', and the device-side Arnoldi loop's fixed K in / out
  if (p->jacobian == PD_JACOBIAN_TIME_AVG) b += (size_t)(kKryM + 4) * total * sizeof(double) + 2 * ns * sizeof(double);
  *bytes = b;
  return PD_OK;
}

int init_impl(const pd_problem* p, int device, void* cuda_stream, pd_handle** out, bool slab);

int paradiag_init(const pd_problem* p, int device, void* cuda_stream, const unsigned char* nccl_id, int rank,
                  int nranks, pd_handle** out) {
  if (!nccl_id && nranks <= 1) return init_impl(p, device, cuda_stream, out, false);
  return shard_init(p, device, cuda_stream, nccl_id, rank, nranks, out);
}

int paradiag_nccl_unique_id(unsigned char id[128]) { return shard_unique_id(id); }

int paradiag_local_rows(const pd_handle* h, int64_t* y0, int64_t* ny_local) {
  if (!h) return fail(PD_EINVAL, "handle is NULL");
  if (h->shard) return shard_local_rows(h, y0, ny_local);
  if (y0) *y0 = 0;
  if (ny_local) *ny_local = h->ny;
  return PD_OK;
}

// internal accessors for shard.cu
pd_shard*& pd_handle_shard(pd_handle* h) { return h->shard; }
cudaStream_t pd_handle_stream(const pd_handle* h) { return h->stream; }
unsigned long long* pd_handle_stats_dev(pd_handle* h) { return &h->st->dmax_bits; }
int pd_set_error(int code, const char* msg) { return fail(code, msg); }

int init_impl(const pd_problem* p, int device, void* cuda_stream, pd_handle** out, bool slab) {
  if (!out) return fail(PD_EINVAL, "out is NULL");
  *out = nullptr;
  int rc = validate(p);
  if (rc) return rc;
  int ndev = 0;
  PD_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(PD_ECUDA, "no such CUDA device");
  PD_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  PD_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    return fail(PD_ECUDA, "libparadiag is built for sm_100a (B200); device is sm_" + std::to_string(prop.major) + std::to_string(prop.minor));

  pd_handle* h = new (std::nothrow) pd_handle();
  if (!h) return fail(PD_ENOMEM, "host allocation");
  h->P = *p;
  h->device = device;
  h->stream = static_cast<cudaStream_t>(cuda_stream);
  geometry(p, &h->nx, &h->ny);
  h->ns = (int64_t)h->nx * h->ny;
  h->total = h->ns * p->nt;
  h->neumann = p->bc == PD_BC_NEUMANN;
  h->log2nt = ilog2(p->nt);
  h->nb = p->nt / 2 + 1;
  h->inv_dt = (double)p->nt / p->t_window;                  // R#20
  h->inv_h2 = (double)p->m * (double)p->m;
  h->b2 = p->beta * p->beta;
  h->e2 = p->eps * p->eps;
  const int M = (int)p->m;
  {
    const char* f = std::getenv("PARADIAG_TLONG");
    const bool force = f && std::atoi(f) != 0;
    h->mixed = !is_pow2(p->nt);          // 2^a 5^b (validate): the mixed-radix four-step passes
    h->tlong = p->nt > kMaxNtShort || h->mixed ||
               (force && p->nt >= 1024 && (p->dim == 2 || (is_pow2(M) && M <= 4096)));
    if (h->mixed) {
      mixed_split(p->nt, &h->n1, &h->n2, h->plan1, &h->nst1, h->plan2, &h->nst2);
      h->log2n1 = h->log2n2 = 0;
    } else {
      tlong_split(h->log2nt, &h->log2n1, &h->log2n2);
      h->n1 = 1 << h->log2n1;
      h->n2 = 1 << h->log2n2;
    }
    h->x1 = h->tlong && p->dim == 1 && (h->nx <= 2 * kX1H || (h->neumann && h->nx == 2 * kX1H + 1));
    if (const char* f3 = std::getenv("PARADIAG_TLFUSE")) h->tlfuse = std::atoi(f3) != 0;
    if (const char* f4 = std::getenv("PARADIAG_MXPAIRS")) h->mxp = std::atoi(f4) == 8 ? 8 : 4;
    if (const char* f5 = std::getenv("PARADIAG_KRYGRAPH")) h->kry_graph = std::atoi(f5) != 0;
    if (const char* f4 = std::getenv("PARADIAG_GRAPH")) h->use_graph = std::atoi(f4) != 0;
    if (const char* f2 = std::getenv("PARADIAG_X1")) h->x1 = h->x1 && std::atoi(f2) != 0;
  }
  h->log2h = (p->dim == 2 || h->tlong) ? ilog2(M) - 1 : 0;
  h->twlog = h->mixed ? std::max(h->log2h, 1) : std::max(h->log2nt, h->log2h);   // mixed: own root tables

  auto cleanup = [&](int code) {
    paradiag_destroy(h);
    return code;
  };
#define PD_TRY(x) do { int rc_ = (x); if (rc_) return cleanup(rc_); } while (0)

  // ---- host tables (closed forms P:156; readings R#1, R#2, R#11)
  const int nt = p->nt;
  std::vector<double> gam(nt), ginv(nt), lam(h->nx);
  std::vector<double2> dl(nt), el(nt), tw(size_t(1) << h->twlog), trig(M + 1);
  const double lna = std::log(p->alpha);
  const double z = std::exp(lna / nt);
  const double spatial_scale = p->dim == 2 ? 1.0 / ((2.0 * M) * (2.0 * M)) : h->tlong ? 1.0 / (2.0 * M) : 1.0;
  for (int j = 0; j < nt; ++j) {
    gam[j] = std::exp(j * lna / nt);
    ginv[j] = std::exp(-j * lna / nt) * (spatial_scale / nt);
  }
  // bins l ≤ N_t/2 from the accurate small angle 2πl/N_t; the upper half as exact conjugates
  // (d_{N-l} = conj d_l): evaluating sin near 2π would carry the argument's absolute rounding
  // (≈ 4e-16) into the small Im d_l of the low bins (1e-12 relative at N_t = 2^15)
  for (int l = 0; l <= nt / 2; ++l) {
    const double ang = 2.0 * M_PI * l / nt;
    dl[l] = make_double2((1.0 - z * std::cos(ang)) * h->inv_dt, (z * std::sin(ang)) * h->inv_dt);
    el[l] = make_double2(p->theta + (1.0 - p->theta) * z * std::cos(ang), -(1.0 - p->theta) * z * std::sin(ang));
    if (l > 0 && l < nt - l) {
      dl[nt - l] = make_double2(dl[l].x, -dl[l].y);
      el[nt - l] = make_double2(el[l].x, -el[l].y);
    }
  }
  for (int i = 0; i < h->nx; ++i) {
    const int pidx = h->neumann ? i : i + 1;
    const double s = std::sin(pidx * M_PI / (2.0 * M));
    lam[i] = -4.0 * h->inv_h2 * s * s;
  }
  const size_t TWN = size_t(1) << h->twlog;
  for (size_t k = 0; k < TWN; ++k) {
    const double ang = 2.0 * M_PI * (double)k / (double)TWN;
    tw[k] = make_double2(std::cos(ang), -std::sin(ang));
  }
  for (int j = 0; j <= M; ++j) trig[j] = make_double2(std::cos(M_PI * j / M), std::sin(M_PI * j / M));
  // k_dtt.cuh split table: (cos, sin)(2πk/M) for k = 32b + j stored at j*E + b, E = M/64
  const int H2 = std::max(M / 2, 1), E2 = std::max(M / 64, 1);
  std::vector<double2> trig2(H2);
  for (int k = 0; k < H2; ++k) {
    const int b = k / 32, j = k % 32;
    trig2[(size_t)j * E2 + b] = trig[std::min(2 * k, M)];
  }
  // k_dtt.cuh pre-processing: (sin, sin)(π(2n, 2n+1)/M), then (cos, cos)(π(2n, 2n+1)/M), n < M/2
  const int HS = std::max(M / 2, 1);
  std::vector<double2> trigsc(2 * (size_t)HS, make_double2(0.0, 0.0));
  for (int n = 0; 2 * n + 1 <= M && n < HS; ++n) {
    trigsc[n] = make_double2(trig[2 * n].y, trig[2 * n + 1].y);
    trigsc[HS + n] = make_double2(trig[2 * n].x, trig[2 * n + 1].x);
  }
  // k_dttp.cuh (M = 2048): k = 16t + j stored at j*64 + t
  std::vector<double2> trig2p(M == 2048 ? 1024 : 0);
  for (int k = 0; k < (int)trig2p.size(); ++k) trig2p[(size_t)(k % 16) * 64 + k / 16] = trig[2 * k];

  // ---- singularity check of d_l + μ (linear kinds): only l = 0 and N_t/2 have real d_l
  if (!is_ch(p->kind)) {
    double worst = INFINITY;
    for (int l : {0, nt / 2}) {
      for (int i = 0; i < h->nx; ++i)
        for (int j = 0; j < (p->dim == 2 ? h->ny : 1); ++j) {
          const double Lam = lam[i] + (p->dim == 2 ? lam[j] : 0.0);
          const double mu = mu_of(p, Lam, h->b2, h->e2);
          const double den = std::hypot(dl[l].x + el[l].x * mu, dl[l].y + el[l].y * mu) /
                             (std::fabs(dl[l].x) + std::fabs(mu) + 1e-300);
          worst = std::min(worst, den);
        }
    }
    if (!(worst > 1e-13)) {
      delete h;
      return fail(PD_ESINGULAR, "shifted system d_l + mu numerically singular (relative " + std::to_string(worst) + ")");
    }
  }

  // ---- device buffers
  // slab mode: caller-owned buffers; k_x1d's workspace rows have an even pitch (pencil pairs)
  if (!slab) PD_TRY(dalloc(h, &h->work, h->x1 ? (size_t)nt * x1_pitch(h) : (size_t)h->total));
  PD_TRY(dalloc(h, &h->u0buf, (size_t)h->ns));
  PD_TRY(dalloc(h, &h->gam, nt));
  PD_TRY(dalloc(h, &h->ginv, nt));
  PD_TRY(dalloc(h, &h->dl, nt));
  if (p->theta != 1.0) PD_TRY(dalloc(h, &h->el, nt));
  std::vector<double2> l3(nt);
  for (int l = 0; l <= nt / 2; ++l) {
    l3[l] = make_double2(z * std::cos(2.0 * M_PI * l / nt), -z * std::sin(2.0 * M_PI * l / nt));
    if (l > 0 && l < nt - l) l3[nt - l] = make_double2(l3[l].x, -l3[l].y);
  }
  if (p->kind == PD_CAHN_HILLIARD_EYRE) PD_TRY(dalloc(h, &h->l3, nt));
  PD_TRY(dalloc(h, &h->lam, h->nx + 1));   // + one finite entry: the pad lines of the column-major wt
  PD_TRY(dalloc(h, &h->tw, TWN));
  PD_TRY(dalloc(h, &h->trig, (size_t)M + 1));
  PD_TRY(dalloc(h, &h->trig2, (size_t)H2));
  PD_TRY(dalloc(h, &h->trigsc, trigsc.size()));
  if (!trig2p.empty()) PD_TRY(dalloc(h, &h->trig2p, trig2p.size()));
  PD_TRY(dalloc(h, &h->st, 1));
  {
    cudaError_t e = cudaMallocHost(&h->st_host, sizeof(DevStats));
    if (e != cudaSuccess) return cleanup(fail(PD_ENOMEM, "cudaMallocHost"));
  }
  if (is_ch(p->kind)) {
    h->njpart = std::max((size_t)((h->nx + kResStrip - 1) / kResStrip) * nt,
                         (size_t)((h->nx + kResTX - 1) / kResTX) * ((h->ny + kResTY - 1) / kResTY) *
                             ((nt + kResChunk - 1) / kResChunk));
    PD_TRY(dalloc(h, &h->jpart, h->njpart));
  }
  if (p->jacobian == PD_JACOBIAN_TIME_AVG) {
    if (p->dim != 2 || slab) return cleanup(fail(PD_EINVAL, "time-averaged Jacobian: 2D, single handle"));
    PD_TRY(dalloc(h, &h->jt, (size_t)h->ns));
    PD_TRY(dalloc(h, &h->wfld, (size_t)h->ns));
    PD_TRY(dalloc(h, &h->kV, (size_t)(kKryM + 1) * (size_t)h->total));
    PD_TRY(dalloc(h, &h->kb, (size_t)h->total));
    PD_TRY(dalloc(h, &h->kpart, (size_t)kKryBlocks * (kKryM + 1)));
    PD_TRY(dalloc(h, &h->kdev, (size_t)kKryM + 2));
    if (cudaMallocHost(&h->khost, (kKryM + 1) * sizeof(double)) != cudaSuccess)
      return cleanup(fail(PD_ENOMEM, "cudaMallocHost"));
    if (const char* f = std::getenv("PARADIAG_CGS_PASSES")) h->cgs_passes = std::max(1, std::min(2, std::atoi(f)));
  }
  auto up = [&](void* d, const void* s, size_t b) { return cudaMemcpyAsync(d, s, b, cudaMemcpyHostToDevice, h->stream); };
  if (up(h->gam, gam.data(), nt * sizeof(double)) || up(h->ginv, ginv.data(), nt * sizeof(double)) ||
      up(h->dl, dl.data(), nt * sizeof(double2)) || (h->el && up(h->el, el.data(), nt * sizeof(double2))) ||
      (h->l3 && up(h->l3, l3.data(), nt * sizeof(double2))) || up(h->lam, lam.data(), h->nx * sizeof(double)) || up(h->lam + h->nx, lam.data() + h->nx - 1, sizeof(double)) ||
      up(h->tw, tw.data(), TWN * sizeof(double2)) || up(h->trig, trig.data(), (M + 1) * sizeof(double2)) ||
      up(h->trig2, trig2.data(), (size_t)H2 * sizeof(double2)) ||
      up(h->trigsc, trigsc.data(), trigsc.size() * sizeof(double2)) ||
      (!trig2p.empty() && up(h->trig2p, trig2p.data(), trig2p.size() * sizeof(double2))))
    return cleanup(fail(PD_ECUDA, "table upload failed"));

  if (h->tlong) {
    // γ_n = α^{n/N_t} (R#2) split at n = N2·n1 + n2; the inverse side carries 1/N_t and the spatial
    // normalisation like ginv
    const int N1 = h->n1, N2 = h->n2;
    std::vector<double> g(2 * (size_t)(N1 + N2));
    for (int i = 0; i < N1; ++i) {
      g[i] = std::exp((double)N2 * i * lna / nt);
      g[N1 + N2 + i] = std::exp(-(double)N2 * i * lna / nt) * (spatial_scale / nt);
    }
    for (int i = 0; i < N2; ++i) {
      g[N1 + i] = std::exp((double)i * lna / nt);
      g[2 * N1 + N2 + i] = std::exp(-(double)i * lna / nt);
    }
    PD_TRY(dalloc(h, &h->tlg, g.size()));
    if (up(h->tlg, g.data(), g.size() * sizeof(double))) return cleanup(fail(PD_ECUDA, "tlong table upload"));
    if (h->mixed) {        // roots of the factor lengths and W_N^b, b < N2 (k_tmix.cuh): exact angles
      std::vector<double2> mt((size_t)N1 + 2 * (size_t)N2);
      auto root = [](int64_t j, int64_t L) {
        const double a = 2.0 * M_PI * (double)j / (double)L;
        return make_double2(std::cos(a), -std::sin(a));
      };
      for (int j = 0; j < N1; ++j) mt[j] = root(j, N1);
      for (int j = 0; j < N2; ++j) mt[(size_t)N1 + j] = root(j, N2);
      for (int j = 0; j < N2; ++j) mt[(size_t)N1 + N2 + j] = root(j, nt);
      PD_TRY(dalloc(h, &h->mtab, mt.size()));
      if (up(h->mtab, mt.data(), mt.size() * sizeof(double2))) return cleanup(fail(PD_ECUDA, "mixed table upload"));
      // digit reversal of the DIF plans (k_tmix.cuh): frequency k = q0 + r0 q1 + … sits at position
      // pos = q0 (L/r0) + q1 (L/(r0 r1)) + …
      std::vector<int> rv(2 * (size_t)(N1 + N2));
      auto rev = [](int L, const int8_t* r, int ns, int* fwd, int* inv) {
        for (int k = 0; k < L; ++k) {
          int kk = k, pos = 0, span = L;
          for (int q = 0; q < ns; ++q) {
            span /= r[q];
            pos += (kk % r[q]) * span;
            kk /= r[q];
          }
          fwd[pos] = k;
          inv[k] = pos;
        }
      };
      rev(N1, h->plan1, h->nst1, rv.data(), rv.data() + N1);
      rev(N2, h->plan2, h->nst2, rv.data() + 2 * N1, rv.data() + 2 * N1 + N2);
      int* drv = nullptr;
      PD_TRY(dalloc(h, &drv, rv.size()));
      if (up(drv, rv.data(), rv.size() * sizeof(int))) return cleanup(fail(PD_ECUDA, "mixed table upload"));
      h->mrev = drv;
    }
    const size_t nc = (size_t)nt * (size_t)((h->ns + 1) / 2);
    PD_TRY(dalloc(h, &h->spec, nc));
    PD_TRY(dalloc(h, &h->w1, nc));
    if (tlong_attrs() != cudaSuccess) return cleanup(fail(PD_ECUDA, "tlong kernel attributes"));
  }
  if (h->x1) {
    // B[0][j][i] = T[2i][j], B[1][j][i] = T[2i+1][j] (k_x1d.cuh even/odd halves): Neumann
    // T[p][j] = c_j cos(π p j/m) (c = 1 at j = 0, m, else 2), hinged T[p][j] = 2 sin(π (p+1)(j+1)/m);
    // angles by the exact integer reduction (p·j) mod 2m
    const int n = h->nx, nh = n / 2, hc = (n + 1) / 2;
    auto Tkj = [&](int k, int j) {
      if (h->neumann) {
        const long a = ((long)k * j) % (2L * M);
        return std::cos(M_PI * (double)a / M) * ((j == 0 || j == M) ? 1.0 : 2.0);
      }
      const long a = ((long)(k + 1) * (j + 1)) % (2L * M);
      return 2.0 * std::sin(M_PI * (double)a / M);
    };
    std::vector<double> B((size_t)2 * kX1K * kX1BP, 0.0);              // [2][kX1K][kX1BP]
    for (int j = 0; j < hc; ++j)
      for (int i = 0; 2 * i < n; ++i) {
        B[(size_t)j * kX1BP + i] = Tkj(2 * i, j);
        if (j < nh && 2 * i + 1 < n) B[(size_t)(kX1K + j) * kX1BP + i] = Tkj(2 * i + 1, j);
      }
    PD_TRY(dalloc(h, &h->x1T, B.size()));
    if (up(h->x1T, B.data(), B.size() * sizeof(double))) return cleanup(fail(PD_ECUDA, "T upload"));
    PD_TRY(allow_smem(k_x1d<0>, kX1Smem));
    PD_TRY(allow_smem(k_x1d<1>, kX1Smem));
    PD_TRY(allow_smem(k_x1d<2>, kX1Smem));
    PD_TRY(allow_smem(k_x1d<3>, kX1Smem));
  }
  if (p->dim == 1 && h->tlong) {
    PD_TRY(allow_smem(k_dtt_rows<1, kLineWarps>, rows_smem(M)));
    PD_TRY(allow_smem(k_dtt_rows<0, kLineWarps>, rows_smem(M)));
    if (const char* f = std::getenv("PARADIAG_FAST")) h->fast = std::atoi(f) != 0;
    PD_TRY(setup_fast_attrs(h));
  } else if (p->dim == 1) {
    const size_t nf = (size_t)h->nx * h->nb;
    PD_TRY(dalloc(h, &h->spec, nf));
    PD_TRY(dalloc(h, &h->w1, nf));
    PD_TRY(dalloc(h, &h->w2, nf));
    PD_TRY(dalloc(h, &h->fac, 4 * nf));
    PD_TRY(dalloc(h, &h->band, 5 * (size_t)h->nx));
    // assembled A = β²D + ε²D² or D² with D = m²·T, T the integer tridiagonal of P:109-118
    const int n = h->nx;
    auto Tij = [&](int i, int j) -> double {
      if (j < 0 || j >= n) return 0.0;
      if (i == j) return -2.0;
      if (std::abs(i - j) != 1) return 0.0;
      if (h->neumann && i == 0 && j == 1) return 2.0;
      if (h->neumann && i == n - 1 && j == n - 2) return 2.0;
      return 1.0;
    };
    std::vector<double> band(5 * (size_t)n);
    const double m2 = h->inv_h2, m4 = m2 * m2;
    for (int i = 0; i < n; ++i)
      for (int k = -2; k <= 2; ++k) {
        const int j = i + k;
        double t2 = 0.0;
        for (int q = i - 1; q <= i + 1; ++q)
          if (q >= 0 && q < n) t2 += Tij(i, q) * Tij(q, j);
        const double t1 = Tij(i, j);
        const double a = p->kind == PD_BIHARMONIC ? m4 * t2 : h->b2 * m2 * t1 + h->e2 * m4 * t2;
        band[(size_t)(k + 2) * n + i] = (j >= 0 && j < n) ? a : 0.0;
      }
    if (up(h->band, band.data(), band.size() * sizeof(double))) return cleanup(fail(PD_ECUDA, "band upload"));
    PentaParams PP;
    PP.n = n; PP.nb = h->nb; PP.neumann = h->neumann; PP.kind = p->kind; PP.inv_h2 = h->inv_h2;
    PP.b2 = h->b2; PP.e2 = h->e2; PP.band = h->band; PP.dl = h->dl; PP.el = h->el;
    PP.l1 = h->fac; PP.l2 = h->fac + nf; PP.iu0 = h->fac + 2 * nf; PP.u1 = h->fac + 3 * nf;
    k_penta_factor<<<(h->nb + 63) / 64, 64, 0, h->stream>>>(PP);
    if (const char* f = std::getenv("PARADIAG_PENTA")) h->penta_cta = std::atoi(f) != 0;
    if (const char* f = std::getenv("PARADIAG_PENTA_REFINE")) h->penta_refine = std::atoi(f);
    if (n <= kPentaCtaMaxN) PD_TRY(allow_smem(k_penta_solve_cta, penta_cta_smem(n)));
    if (cudaGetLastError() != cudaSuccess) return cleanup(fail(PD_ECUDA, "penta factor launch"));
    if (time_smem(nt, kTime1DWarps) <= kSmemMax) {
      PD_TRY(allow_smem(k_time_fwd_1d<kTime1DWarps>, time_smem(nt, kTime1DWarps)));
      PD_TRY(allow_smem(k_time_inv_1d<kTime1DWarps>, time_smem(nt, kTime1DWarps)));
    } else {
      PD_TRY(allow_smem(k_time_fwd_1d<1>, time_smem(nt, 1)));
      PD_TRY(allow_smem(k_time_inv_1d<1>, time_smem(nt, 1)));
    }
  } else {
    if (h->tlong) {
    } else if (time_smem(nt, kTimeWarps) <= kSmemMax) {
      PD_TRY(allow_smem(k_time_solve_2d<kTimeWarps>, time_smem(nt, kTimeWarps)));
    } else {
      PD_TRY(allow_smem(k_time_solve_2d<1>, time_smem(nt, 1)));
    }
    PD_TRY(allow_smem(k_dtt_rows<1, kLineWarps>, rows_smem(M)));
    PD_TRY(allow_smem(k_dtt_rows<0, kLineWarps>, rows_smem(M)));
    if (cols_per_cta(M) == kColW) {
      PD_TRY(allow_smem(k_dtt_cols<1, kColW>, cols_smem(M)));
      PD_TRY(allow_smem(k_dtt_cols<0, kColW>, cols_smem(M)));
    } else {
      PD_TRY(allow_smem(k_dtt_cols<1, 4>, cols_smem(M, 4)));
      PD_TRY(allow_smem(k_dtt_cols<0, 4>, cols_smem(M, 4)));
    }
    PD_TRY(allow_smem(k_residual_tile<0>, kResSmem));
    PD_TRY(allow_smem((k_residual_tile<0, false, 1>), kResSmem));
    PD_TRY(allow_smem((k_residual_tile<0, false, 1, true>), kResSmem));
    PD_TRY(allow_smem((k_residual_tile<0, false, 2>), kResSmem));
    PD_TRY(allow_smem((k_residual_tile<0, false, 3>), kResSmem));
    PD_TRY(allow_smem((k_residual_tile<1, false, 1>), kResSmem));
    PD_TRY(allow_smem((k_residual_tile<2, false, 2>), kResSmem));
    PD_TRY(allow_smem(k_residual_tile<0, true>, kResSmemUpd));
    PD_TRY(allow_smem((k_residual_tile<0, true, 1>), kResSmemUpd));
    PD_TRY(allow_smem(k_residual_tile<1, true>, kResSmemUpd));
    if (const char* f = std::getenv("PARADIAG_PIPELINE")) h->pipe = std::atoi(f) != 0;
    if (can_pipeline(h)) {              // the pipelined solve's second iterate / workspace buffers
      PD_TRY(dalloc(h, &h->Ub, (size_t)h->total));
      PD_TRY(dalloc(h, &h->work2, (size_t)h->total));
    }
    if (const char* f = std::getenv("PARADIAG_FAST")) h->fast = std::atoi(f) != 0;
    if (const char* f = std::getenv("PARADIAG_DTT")) h->dtt_ver = std::atoi(f) == 4 ? 4 : 3;
    if (const char* f = std::getenv("PARADIAG_TMA")) h->tma = std::atoi(f) != 0;
    if (const char* f = std::getenv("PARADIAG_TUNE")) h->tune = std::atoi(f);
    if (const char* f = std::getenv("PARADIAG_STAGGER")) h->stagger_ns = std::atoi(f);
    PD_TRY(setup_fast_attrs(h));
    if (h->tma && h->fast && !slab && !h->tlong && nt >= 32 && nt <= 512 && p->m >= 64 && p->m <= 2048) {
      h->lp = (h->ny + 1) & ~(int64_t)1;        // column-major lines, 16-byte aligned
      h->ps = (int64_t)h->nx * h->lp;
      PD_TRY(dalloc(h, &h->wt, (size_t)nt * h->ps));
      // the pad column shares a complex pencil with point ns-1 in the time pass: keep it finite
      if (cudaMemsetAsync(h->wt, 0, (size_t)nt * h->ps * sizeof(double), h->stream) != cudaSuccess)
        return cleanup(fail(PD_ECUDA, "wt memset"));
      const char* fw = std::getenv("PARADIAG_WP");
      // default for M = 2048 (y⁻¹ 13.4 -> 10.4 ms on c5); M = 512 / 1024 only with PARADIAG_WP=1 (c3:
      // y⁻¹ 0.231 -> 0.244 ms — its 32-column tiles already store 256-byte row segments)
      const bool wp_on = fw ? std::atoi(fw) != 0 : p->m == 2048;
      if ((p->m == 512 || p->m == 1024 || p->m == 2048) && h->dtt_ver == 3 && wp_on) {
        h->lpx = (h->nx + 7) & ~(int64_t)7;
        PD_TRY(dalloc(h, &h->wp, (size_t)nt * h->ny * h->lpx));
        const unsigned cw = 8u * 2048u / (unsigned)p->m;            // tile columns (8 / 16 / 32)
        if (!make_map_3d(&h->wp_map, h->wp, h->nx, h->ny, nt, h->lpx, cw, kYsRows * 8 / cw))
          return cleanup(fail(PD_ECUDA, "wp tensor map encode failed"));
      }
    }
  }
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return cleanup(fail(PD_ECUDA, "init synchronize"));
#undef PD_TRY
  *out = h;
  return PD_OK;
}

int paradiag_residual(pd_handle* h, const double* u0, const double* U, double* r, double* jbar_out) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (h->shard) return fail(PD_EINVAL, "residual: single-GPU handles only (sharded ranks need the halo exchange)");
  if (!u0 || !U || !r) return fail(PD_EINVAL, "NULL buffer");
  if (r == U) return fail(PD_EINVAL, "r must not alias U");
  if ((rc = launch_residual(h, u0, U, r))) return rc;
  if (jbar_out) {
    PD_CUDA(cudaMemcpyAsync(h->st_host, h->st, sizeof(DevStats), cudaMemcpyDeviceToHost, h->stream));
    PD_CUDA(cudaStreamSynchronize(h->stream));
    *jbar_out = is_ch(h->P.kind) ? h->st_host->jbar : 0.0;
  }
  return PD_OK;
}

int paradiag_apply_precond(pd_handle* h, const double* r, double* delta, double jbar) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!r || !delta) return fail(PD_EINVAL, "NULL buffer");
  if (h->shard) return shard_apply_precond(h, r, delta);
  if (is_ch(h->P.kind)) {
    k_set_jbar<<<1, 1, 0, h->stream>>>(h->st, jbar);
    PD_LAUNCHED();
  }
  k_reset_stats<<<1, 1, 0, h->stream>>>(h->st);
  PD_LAUNCHED();
  return precond(h, r, delta);
}

int paradiag_apply_precond_jt(pd_handle* h, const double* r, double* delta, const double* jt) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!r || !delta || !jt) return fail(PD_EINVAL, "NULL buffer");
  if (h->P.jacobian != PD_JACOBIAN_TIME_AVG || !h->kV)
    return fail(PD_EINVAL, "handle was not initialised with jacobian = PD_JACOBIAN_TIME_AVG");
  k_reset_stats<<<1, 1, 0, h->stream>>>(h->st);
  PD_LAUNCHED();
  if ((rc = setup_wprime(h, jt))) return rc;
  return precond_jt(h, r, delta);
}

int paradiag_iterate(pd_handle* h, const double* u0, double* U, pd_iter_info* info) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!u0 || !U || !info) return fail(PD_EINVAL, "NULL argument");
  if (h->shard) return shard_iterate(h, u0, U, info);
  if (reinterpret_cast<uintptr_t>(U) % 16) return fail(PD_EINVAL, "U must be 16-byte aligned");
  pd_iter_info tmp = *info;
  rc = iteration(h, u0, U, &tmp);
  tmp.iters = info->iters + 1;
  tmp.converged = (h->P.fixed_iters <= 0) && tmp.delta_max <= h->P.tol * tmp.u_max;
  tmp.growth = (info->iters > 0 && tmp.delta_max > info->delta_max) ? info->growth + 1 : 0;   // PD_GROWTH_LIMIT
  *info = tmp;
  return rc;
}

int paradiag_solve(pd_handle* h, const double* u0, double* U, pd_solve_info* info) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!u0 || !U || !info) return fail(PD_EINVAL, "NULL argument");
  if (h->shard) return shard_solve(h, u0, U, info);
  if (reinterpret_cast<uintptr_t>(U) % 16) return fail(PD_EINVAL, "U must be 16-byte aligned");
  const auto t0 = std::chrono::steady_clock::now();
  std::memset(info, 0, sizeof(*info));
  const double* cur_u0 = u0;
  int status = PD_OK;
  bool all_conv = true;
  for (int w = 0; w < h->P.n_windows; ++w) {
    if (can_pipeline(h)) {
      int iters = 0;
      bool conv = false, div = false;
      double rel = 0.0;
      if ((rc = solve_window_pipelined(h, cur_u0, U, &iters, &conv, &rel, &div))) {
        info->windows_done = w;
        return rc;
      }
      info->iters[w] = iters;
      info->last_rel[w] = rel;
      info->diverging += div ? 1 : 0;
      info->windows_done = w + 1;
      all_conv = all_conv && conv;
      if (!conv && h->P.fixed_iters <= 0) status = PD_NOT_CONVERGED;
      if (w + 1 < h->P.n_windows) {
        PD_CUDA(cudaMemcpyAsync(h->u0buf, U + (size_t)(h->P.nt - 1) * h->ns, h->ns * sizeof(double),
                                cudaMemcpyDeviceToDevice, h->stream));
        cur_u0 = h->u0buf;
      }
      continue;
    }
    if (graph_ok(h)) {                 // device-side loop: one graph launch per window
      if (cur_u0 != h->u0buf) {
        PD_CUDA(cudaMemcpyAsync(h->u0buf, cur_u0, h->ns * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
        cur_u0 = h->u0buf;
      }
      if ((!h->gexec || h->gU != U) && build_graph(h, U) != PD_OK) {
        h->use_graph = false;            // capture unsupported here: host loop from now on
        cudaGetLastError();
      }
    }
    if (graph_ok(h) && h->gexec && h->gU == U) {
      if ((rc = init_iterate(h, U, cur_u0))) return rc;
      int iters = 0;
      bool conv = false, div = false;
      double rel = 0.0;
      rc = graph_window(h, &iters, &conv, &rel, &div);
      info->iters[w] = iters;
      info->last_rel[w] = rel;
      info->diverging += div ? 1 : 0;
      if (rc) {
        info->windows_done = w;
        return rc;
      }
      info->windows_done = w + 1;
      all_conv = all_conv && conv;
      if (!conv && h->P.fixed_iters <= 0) status = PD_NOT_CONVERGED;
      if (w + 1 < h->P.n_windows) {    // hand-off: u0 ← U_{N_t}
        PD_CUDA(cudaMemcpyAsync(h->u0buf, U + (size_t)(h->P.nt - 1) * h->ns, h->ns * sizeof(double),
                                cudaMemcpyDeviceToDevice, h->stream));
        cur_u0 = h->u0buf;
      }
      continue;
    }
    if ((rc = init_iterate(h, U, cur_u0))) return rc;
    const int kmax = h->P.fixed_iters > 0 ? h->P.fixed_iters : h->P.max_iter;
    bool conv = false, div = false;
    int k = 0, growth = 0;
    double dprev = 0.0;
    pd_iter_info it{};
    for (k = 1; k <= kmax; ++k) {
      if ((rc = iteration(h, cur_u0, U, &it))) {
        info->iters[w] = k;
        info->windows_done = w;
        return rc;
      }
      if (h->P.fixed_iters <= 0 && it.delta_max <= h->P.tol * it.u_max) {
        conv = true;
        break;
      }
      growth = (k > 1 && it.delta_max > dprev) ? growth + 1 : 0;       // SURVEY §5.3 (PD_GROWTH_LIMIT)
      dprev = it.delta_max;
      if (growth >= PD_GROWTH_LIMIT) {
        div = true;
        if (h->P.fixed_iters <= 0) break;
      }
    }
    info->diverging += div ? 1 : 0;
    info->iters[w] = std::min(k, kmax);
    info->last_rel[w] = it.rel;
    info->windows_done = w + 1;
    all_conv = all_conv && conv;
    if (!conv && h->P.fixed_iters <= 0) status = PD_NOT_CONVERGED;
    if (w + 1 < h->P.n_windows) {      // hand-off: u0 ← U_{N_t}
      PD_CUDA(cudaMemcpyAsync(h->u0buf, U + (size_t)(h->P.nt - 1) * h->ns, h->ns * sizeof(double),
                              cudaMemcpyDeviceToDevice, h->stream));
      cur_u0 = h->u0buf;
    }
  }
  info->converged = h->P.fixed_iters > 0 ? 0 : (all_conv ? 1 : 0);
  PD_CUDA(cudaStreamSynchronize(h->stream));
  info->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return status;
}

int paradiag_solve_host(pd_handle* h, const double* u0_host, double* uT_host, pd_solve_info* info) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (h->shard) return fail(PD_EINVAL, "solve_host: single-GPU handles only (a sharded rank owns device slabs)");
  if (!u0_host || !uT_host || !info) return fail(PD_EINVAL, "NULL argument");
  if (!h->Uint && (rc = dalloc(h, &h->Uint, (size_t)h->total))) return rc;
  // window 1's u0 is staged in the hand-off buffer; it is only overwritten after window 1 ends
  double* d_u0 = h->u0buf;
  PD_CUDA(cudaMemcpyAsync(d_u0, u0_host, h->ns * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  rc = paradiag_solve(h, d_u0, h->Uint, info);
  if (rc < 0) return rc;
  PD_CUDA(cudaMemcpyAsync(uT_host, h->Uint + (size_t)(h->P.nt - 1) * h->ns, h->ns * sizeof(double),
                          cudaMemcpyDeviceToHost, h->stream));
  PD_CUDA(cudaStreamSynchronize(h->stream));
  return rc;
}

int paradiag_launches_per_iteration(const pd_handle* h) {
  if (!h) return 0;
  if (h->P.jacobian == PD_JACOBIAN_TIME_AVG) return -1;   // data dependent (inner GMRES steps)
  const int ntime = h->tlong ? (h->tlfuse && (h->mixed || (h->log2n2 == 10 && h->log2n1 >= 5)) ? 3 : 5) : 1;
  if (h->x1) return 1 /*reset*/ + 1 /*residual + x*/ + ntime + 1 /*x⁻¹ + update*/;
  int n = 1 /*reset*/ + 1 /*residual*/ + (can_fuse_update(h) ? 0 : 1) /*update*/;
  n += h->P.dim == 2 ? 4 + ntime : (h->tlong ? 2 + ntime : 3);
  if (is_ch(h->P.kind)) n += 1;
  return n;
}

int paradiag_profile(pd_handle* h, int enable) {
  if (!h) return fail(PD_EINVAL, "handle is NULL");
  h->prof = enable != 0;
  for (int i = 0; i < PD_NKERNELS; ++i) {
    h->prof_ms[i] = 0.0;
    h->prof_n[i] = 0;
    h->ev_used[i] = false;
  }
  return PD_OK;
}

int paradiag_profile_read(const pd_handle* h, pd_kernel_time* out, int max_entries, int* n_out) {
  if (!h || !n_out) return fail(PD_EINVAL, "NULL argument");
  int n = 0;
  for (int i = 0; i < PD_NKERNELS; ++i) {
    if (!h->prof_n[i]) continue;
    if (out && n < max_entries) {
      std::memset(&out[n], 0, sizeof(pd_kernel_time));
      std::strncpy(out[n].name, kKernelNames[i], sizeof(out[n].name) - 1);
      out[n].launches = h->prof_n[i];
      out[n].total_ms = h->prof_ms[i];
    }
    ++n;
  }
  *n_out = n;
  return PD_OK;
}

// ----------------------------------------------------------------------------- slab mode
int paradiag_init_slab(const pd_problem* p, int device, void* cuda_stream, int64_t y0, int64_t nyl, int64_t x0,
                       int64_t nxl, pd_handle** out) {
  if (!out) return fail(PD_EINVAL, "out is NULL");
  *out = nullptr;
  int rc = validate(p);
  if (rc) return rc;
  if (p->dim != 2 || is_ch(p->kind) || p->theta != 1.0)
    return fail(PD_EINVAL, "slab mode: 2D linear kinds with theta = 1 (CH runs as replicas, DESIGN.md §8)");
  if (p->m < 64 || p->m > 2048 || p->nt < 32 || p->nt > 1024)
    return fail(PD_EINVAL, "slab mode: needs the register-FFT sizes (64 <= m <= 2048, 32 <= nt <= 1024)");
  int nx, ny;
  geometry(p, &nx, &ny);
  if (y0 < 0 || nyl < 3 || y0 + nyl > ny || x0 < 0 || nxl < 1 || x0 + nxl > nx)
    return fail(PD_EINVAL, "slab mode: row slab needs >= 3 rows and both slabs inside the grid");
  // a single-GPU handle of the same problem provides the tables; its iterate-sized workspace is
  // not allocated in slab mode (the caller owns every buffer)
  pd_problem q = *p;
  rc = init_impl(&q, device, cuda_stream, out, true);
  if (rc) return rc;
  pd_handle* h = *out;
  h->slab = true;
  h->y0 = (int)y0; h->nyl = (int)nyl; h->x0 = (int)x0; h->nxl = (int)nxl;
  return PD_OK;
}

int paradiag_slab_geometry(const pd_handle* h, int64_t* y0, int64_t* nyl, int64_t* x0, int64_t* nxl) {
  if (!h || !h->slab) return fail(PD_EINVAL, "not a slab handle");
  if (y0) *y0 = h->y0;
  if (nyl) *nyl = h->nyl;
  if (x0) *x0 = h->x0;
  if (nxl) *nxl = h->nxl;
  return PD_OK;
}

int paradiag_slab_residual(pd_handle* h, const double* u0_l, const double* U_l, const double* halo_lo,
                           const double* halo_hi, double* r_l) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!h->slab) return fail(PD_EINVAL, "not a slab handle");
  if (!u0_l || !U_l || !r_l) return fail(PD_EINVAL, "NULL buffer");
  if ((h->y0 > 0 && !halo_lo) || (h->y0 + h->nyl < h->ny && !halo_hi))
    return fail(PD_EINVAL, "interior slab edges need halo rows");
  ResidualParams R;
  R.nx = h->nx; R.ny = h->nyl; R.nt = h->P.nt; R.dim = 2;
  R.neumann = h->neumann; R.kind = h->P.kind;
  R.inv_h2 = h->inv_h2; R.inv_dt = h->inv_dt; R.b2 = h->b2; R.e2 = h->e2;
  R.y0g = h->y0; R.nyg = h->ny; R.hlo = halo_lo; R.hhi = halo_hi; R.theta = 1.0;
  prof_begin(h, K_RESIDUAL);
  dim3 grd((h->nx + kResTX - 1) / kResTX, (h->nyl + kResTY - 1) / kResTY, (h->P.nt + kResChunk - 1) / kResChunk);
  // slab handles are linear kinds with θ = 1 (init_slab): the variant without the CH branch
  if (is_ch(h->P.kind)) k_residual_tile<0><<<grd, kResThreads, kResSmem, h->stream>>>(u0_l, U_l, r_l, R, h->jpart);
  else k_residual_tile<0, false, 3><<<grd, kResThreads, kResSmem, h->stream>>>(u0_l, U_l, r_l, R, h->jpart);
  prof_end(h, K_RESIDUAL);
  PD_LAUNCHED();
  return PD_OK;
}

int paradiag_slab_xrange(pd_handle* h, const double* in, double* out, int want_dmax, const int64_t* seg_in,
                         const int64_t* seg_out, int64_t n0, int64_t nn);
int paradiag_slab_yrange(pd_handle* h, const double* in, double* cols, double* out, int stage, const int64_t* seg,
                         int64_t n0, int64_t nn);

int paradiag_slab_xpass(pd_handle* h, const double* in, double* out, int want_dmax) {
  return paradiag_slab_xrange(h, in, out, want_dmax, nullptr, nullptr, 0, h ? h->P.nt : 0);
}

int paradiag_slab_ypass(pd_handle* h, double* buf) {
  return paradiag_slab_ypass_seg(h, buf, buf, buf, nullptr, nullptr);
}

int paradiag_slab_xpass_seg(pd_handle* h, const double* in, double* out, int want_dmax, const int64_t* seg_in,
                            const int64_t* seg_out) {
  return paradiag_slab_xrange(h, in, out, want_dmax, seg_in, seg_out, 0, h ? h->P.nt : 0);
}

int paradiag_slab_ypass_seg(pd_handle* h, const double* in, double* cols, double* out, const int64_t* seg_in,
                            const int64_t* seg_out) {
  const int64_t nt = h ? h->P.nt : 0;
  int rc;
  if ((rc = paradiag_slab_yrange(h, in, cols, cols, 0, seg_in, 0, nt))) return rc;
  if ((rc = paradiag_slab_yrange(h, cols, cols, cols, 1, nullptr, 0, nt))) return rc;
  return paradiag_slab_yrange(h, cols, cols, out, 2, seg_out, 0, nt);
}

}  // extern "C"

namespace {
// {k, (e0, cnt, off) × k} → SegMap; checks that the blocks tile [0, nel) in order
int read_segmap(const int64_t* d, int nel, SegMap* S) {
  S->n = 0;
  if (!d) return PD_OK;
  const int64_t k = d[0];
  if (k < 1 || k > kMaxSeg) return fail(PD_EINVAL, "segment map: 1..8 blocks");
  int64_t next = 0;
  for (int q = 0; q < k; ++q) {
    const int64_t e0 = d[1 + 3 * q], cnt = d[2 + 3 * q], off = d[3 + 3 * q];
    // off may be negative: a peer's buffer mapped into this address space (CUDA IPC / one device)
    // is addressed as an element offset from this call's buffer pointer
    if (e0 != next || cnt < 0) return fail(PD_EINVAL, "segment map: blocks must tile the line in order");
    S->e0[q] = (int)e0;
    S->cnt[q] = (int)cnt;
    S->off[q] = off;
    next = e0 + cnt;
  }
  if (next != nel) return fail(PD_EINVAL, "segment map: blocks must cover the whole line");
  // empty trailing blocks are skipped by the kernels' loops; the first block may not be empty
  // for the column kernels' running block index, so drop leading empty blocks
  int q0 = 0;
  while (q0 < k && S->cnt[q0] == 0) ++q0;
  if (q0) {
    for (int q = q0; q < k; ++q) {
      S->e0[q - q0] = S->e0[q];
      S->cnt[q - q0] = S->cnt[q];
      S->off[q - q0] = S->off[q];
    }
  }
  S->n = (int)k - q0;
  return PD_OK;
}

// one block covering the whole line is the plain layout shifted by its offset
int64_t plain_shift(SegMap* S) {
  if (S->n != 1) return 0;
  S->n = 0;
  return S->off[0];
}
}  // namespace

extern "C" {

int paradiag_slab_xrange(pd_handle* h, const double* in, double* out, int want_dmax, const int64_t* seg_in,
                         const int64_t* seg_out, int64_t n0, int64_t nn) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!h->slab) return fail(PD_EINVAL, "not a slab handle");
  if (!in || !out) return fail(PD_EINVAL, "NULL buffer");
  if (n0 < 0 || nn < 1 || n0 + nn > h->P.nt) return fail(PD_EINVAL, "slice range outside [0, nt)");
  LineParams L = line_params(h, 0, want_dmax ? &h->st->dmax_bits : nullptr);
  L.nlines = nn * h->nyl;
  if ((rc = read_segmap(seg_in, h->nx, &L.sin)) || (rc = read_segmap(seg_out, h->nx, &L.sout))) return rc;
  // slab-layout buffers start at slice n0; block buffers are addressed relative to the range
  const int64_t slice = (int64_t)h->nyl * h->nx;
  in += seg_in ? plain_shift(&L.sin) : n0 * slice;
  out += seg_out ? plain_shift(&L.sout) : n0 * slice;
  const int ver = h->dtt_ver;
  h->dtt_ver = 3;                                   // the block addressing lives in the v3 kernels
  prof_begin(h, want_dmax ? K_XINV : K_XFWD);
  const bool ok = fast_line_any(h, in, out, 0, L);
  prof_end(h, want_dmax ? K_XINV : K_XFWD);
  h->dtt_ver = ver;
  if (!ok) return fail(PD_EINVAL, "slab mode: unsupported line length");
  PD_LAUNCHED();
  return PD_OK;
}

int paradiag_slab_yrange(pd_handle* h, const double* in, double* cols, double* out, int stage, const int64_t* seg,
                         int64_t n0, int64_t nn) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!h->slab) return fail(PD_EINVAL, "not a slab handle");
  if (!in || !cols || !out) return fail(PD_EINVAL, "NULL buffer");
  if (stage < 0 || stage > 2) return fail(PD_EINVAL, "stage: 0 y-DTT, 1 time pass, 2 y-DTT inverse");
  if (stage != 1 && (n0 < 0 || nn < 1 || n0 + nn > h->P.nt)) return fail(PD_EINVAL, "slice range outside [0, nt)");
  const int64_t slice = (int64_t)h->ny * h->nxl;     // column slab [nt][ny][nxl]: lines along y, stride nxl
  FastLaunch F = fast_launch(h);
  F.nx = h->nxl;
  F.ns = slice;
  F.dtt_ver = 3;                                    // the block addressing lives in the v3 kernels
  if (stage == 1) {
    TimeParams T = time_params(h, nullptr);
    T.ns = slice;
    T.nx = h->nxl;
    T.xoff = h->x0;
    T.gamma_folded = 1;
    prof_begin(h, K_TIME);
    switch (h->P.nt) {
      case 32: fast_time<1>(cols, cols, T, F); break;
      case 64: fast_time<2>(cols, cols, T, F); break;
      case 128: fast_time<4>(cols, cols, T, F); break;
      case 256: fast_time<8>(cols, cols, T, F); break;
      case 512: fast_time<16>(cols, cols, T, F); break;
      default: fast_time<32>(cols, cols, T, F); break;
    }
    prof_end(h, K_TIME);
    PD_LAUNCHED();
    return PD_OK;
  }
  LineParams L = line_params(h, 1, nullptr);
  L.nlines = nn * h->nxl;
  L.nx = h->nxl;
  L.ns = slice;
  L.ps_in = L.ps_out = L.ns;
  L.nel = h->ny;
  F.nt = (int)nn;
  SegMap S;
  if ((rc = read_segmap(seg, h->ny, &S))) return rc;
  const int64_t shift = seg ? plain_shift(&S) : n0 * slice;
  const double* src;
  double* dst;
  int kid;
  if (stage == 0) {                                 // y forward: blocks (or the slab) → cols
    L.sin = S;
    src = in + shift;
    dst = cols + n0 * slice;
    L.oscale = h->gam + n0;                         // Γ_α folded into the forward y outputs
    kid = K_YFWD;
  } else {                                          // y inverse: cols → blocks (or the slab)
    L.sout = S;
    src = cols + n0 * slice;
    dst = out + shift;
    L.oscale = h->ginv + n0;
    kid = K_YINV;
  }
  const int nm = h->neumann ? 1 : 0;
  prof_begin(h, kid);
  switch (L.M) {
    case 64: fast_line<1>(nm, 1, src, dst, L, F); break;
    case 128: fast_line<2>(nm, 1, src, dst, L, F); break;
    case 256: fast_line<4>(nm, 1, src, dst, L, F); break;
    case 512: fast_line<8>(nm, 1, src, dst, L, F); break;
    case 1024: fast_line<16>(nm, 1, src, dst, L, F); break;
    default: fast_line<32>(nm, 1, src, dst, L, F); break;
  }
  prof_end(h, kid);
  PD_LAUNCHED();
  return PD_OK;
}

int paradiag_ipc_handle(const void* dev_ptr, unsigned char handle[64]) {
  if (!dev_ptr || !handle) return fail(PD_EINVAL, "NULL argument");
  cudaIpcMemHandle_t hd;
  PD_CUDA(cudaIpcGetMemHandle(&hd, const_cast<void*>(dev_ptr)));
  static_assert(sizeof(hd) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle, &hd, 64);
  return PD_OK;
}

int paradiag_ipc_open(const unsigned char handle[64], void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(PD_EINVAL, "NULL argument");
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle, 64);
  PD_CUDA(cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess));
  return PD_OK;
}

int paradiag_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return fail(PD_EINVAL, "NULL argument");
  PD_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return PD_OK;
}

int paradiag_slab_update_range(pd_handle* h, double* U_l, const double* delta_l, int64_t n0, int64_t nn) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!h->slab) return fail(PD_EINVAL, "not a slab handle");
  if (!U_l || !delta_l) return fail(PD_EINVAL, "NULL buffer");
  if (n0 < 0 || nn < 1 || n0 + nn > h->P.nt) return fail(PD_EINVAL, "slice range outside [0, nt)");
  const int64_t slice = (int64_t)h->nyl * h->nx;
  prof_begin(h, K_UPDATE);
  k_update<<<148 * 8, 256, 0, h->stream>>>(U_l + n0 * slice, delta_l + n0 * slice, (size_t)(nn * slice), h->st, 0,
                                           1.0, 1.0);
  prof_end(h, K_UPDATE);
  PD_LAUNCHED();
  return PD_OK;
}

int paradiag_slab_update(pd_handle* h, double* U_l, const double* delta_l) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!h->slab) return fail(PD_EINVAL, "not a slab handle");
  if (!U_l || !delta_l) return fail(PD_EINVAL, "NULL buffer");
  prof_begin(h, K_UPDATE);
  k_update<<<148 * 8, 256, 0, h->stream>>>(U_l, delta_l, (size_t)h->P.nt * h->nyl * h->nx, h->st, 0, 1.0, 1.0);
  prof_end(h, K_UPDATE);
  PD_LAUNCHED();
  return PD_OK;
}

// ---- time slabs (1D long windows across ranks): contiguous time rows per rank for
// the residual / x transforms / update, column (x-mode) blocks of all N_t rows for the time pass
namespace {
int tslab_check(pd_handle* h, int64_t bcols) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!h->x1 || !h->tlong || is_ch(h->P.kind) || h->P.jacobian != PD_JACOBIAN_SCALAR)
    return fail(PD_EINVAL, "time slabs need a 1D linear long-window handle with N_x <= 64 (DMMA x transforms)");
  const int64_t pitch = x1_pitch(h);
  if (bcols <= 0 || (bcols & 1) || pitch % bcols) return fail(PD_EINVAL, "bcols must be even and divide the mode pitch");
  return PD_OK;
}
}  // namespace

int paradiag_tslab_pitch(const pd_handle* h, int64_t* pitch) {
  if (!h || !pitch) return PD_EINVAL;
  *pitch = h->x1 ? (int64_t)x1_pitch(h) : 0;
  return PD_OK;
}

int paradiag_tslab_residual(pd_handle* h, const double* u_prev, const double* U_l, int64_t nn, double* blocks,
                            int64_t bcols) {
  int rc = tslab_check(h, bcols);
  if (rc) return rc;
  if (!u_prev || !U_l || !blocks) return fail(PD_EINVAL, "NULL buffer");
  if (nn < 1 || nn > h->P.nt) return fail(PD_EINVAL, "row count out of range");
  return launch_x1d(h, 0, u_prev, U_l, blocks, K_XRES, nn, (int)bcols);
}

int paradiag_tslab_time(pd_handle* h, double* cols, int64_t c0, int64_t bcols) {
  int rc = tslab_check(h, bcols);
  if (rc) return rc;
  if (!cols) return fail(PD_EINVAL, "NULL buffer");
  if (c0 < 0 || c0 % bcols || c0 >= x1_pitch(h)) return fail(PD_EINVAL, "c0 must be a block start inside the pitch");
  if (c0 >= h->ns) return PD_OK;                 // a block of padding only: nothing to solve
  return tlong_time(h, cols, cols, c0, bcols);
}

int paradiag_tslab_update(pd_handle* h, const double* blocks, int64_t bcols, double* U_l, int64_t nn) {
  int rc = tslab_check(h, bcols);
  if (rc) return rc;
  if (!blocks || !U_l) return fail(PD_EINVAL, "NULL buffer");
  if (nn < 1 || nn > h->P.nt) return fail(PD_EINVAL, "row count out of range");
  return launch_x1d(h, 3, nullptr, blocks, U_l, K_XUPD, nn, (int)bcols);
}

int paradiag_copy3d(pd_handle* h, const double* src, double* dst, int64_t n0, int64_t n1, int64_t n2, int64_t s0,
                    int64_t s1, int64_t d0, int64_t d1) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (n0 <= 0 || n1 <= 0 || n2 <= 0) return PD_OK;
  if (!src || !dst) return fail(PD_EINVAL, "NULL buffer");
  const int64_t rows = n0 * n1;
  const unsigned grid = (unsigned)std::min<int64_t>(rows, 148 * 16);
  k_copy3d<<<grid, 256, 0, h->stream>>>(src, dst, n0, n1, n2, s0, s1, d0, d1);
  PD_LAUNCHED();
  return PD_OK;
}

int paradiag_stats_reset(pd_handle* h) {
  int rc = check_handle(h);
  if (rc) return rc;
  k_reset_stats<<<1, 1, 0, h->stream>>>(h->st);
  PD_LAUNCHED();
  return PD_OK;
}

int paradiag_stats_read(pd_handle* h, double* dmax, double* umax) {
  int rc = check_handle(h);
  if (rc) return rc;
  PD_CUDA(cudaMemcpyAsync(h->st_host, h->st, sizeof(DevStats), cudaMemcpyDeviceToHost, h->stream));
  PD_CUDA(cudaStreamSynchronize(h->stream));
  prof_collect(h);
  if (dmax) std::memcpy(dmax, &h->st_host->dmax_bits, sizeof(double));
  if (umax) std::memcpy(umax, &h->st_host->umax_bits, sizeof(double));
  return PD_OK;
}

void paradiag_destroy(pd_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->shard) shard_destroy(h->shard);
  for (int i = 0; i < PD_NKERNELS; ++i)
    for (int j = 0; j < 2; ++j)
      if (h->ev[i][j]) cudaEventDestroy(h->ev[i][j]);
  for (void* q : h->allocs) cudaFree(q);
  if (h->st_host) cudaFreeHost(h->st_host);
  if (h->khost) cudaFreeHost(h->khost);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->graph) cudaGraphDestroy(h->graph);
  if (h->kgexec) cudaGraphExecDestroy(h->kgexec);
  if (h->kgraph) cudaGraphDestroy(h->kgraph);
  if (h->kd_host) cudaFreeHost(h->kd_host);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  if (h->ctl_host) cudaFreeHost(h->ctl_host);
  delete h;
}

}  // extern "C"
