// k_krylov.cuh — NEXT-4: Step-(2) with the paper's time-only averaged Jacobian.
// J̃ = I_t ⊗ (1/N_t) Σ_n J_s(u_n) = diag(jt) is spatially varying, so Step-(2) is no longer a
// per-mode divide.  The engine solves G̃' δ = r in the time domain by restarted GMRES, left-
// preconditioned by the scalar-J̄ P_α⁻¹ (the spectral pipeline):
//   G̃' = P(J̄) - I_t ⊗ Δ_h diag(w'),   w' = jt - c - J̄,   J̄ = mean(jt) - c,
// c = 1 for PinT-I (-Δ_h J̃ + Δ_h) and 0 for PinT-II, so each Krylov step applies
// K x = P⁻¹ Δ_h(w' ⊙ x).  The kernels here are the vector pieces: the time mean of 3U², w' and J̄,
// the variable-coefficient Laplacian, and deterministic multi-vector dots / updates (fixed block
// partition and fixed-order sums, so two runs give the same bits).
#pragma once
#include "common.cuh"

namespace pd {

constexpr int kKryBlocks = 592;          // 4 × 148: fixed partition of the dot products
constexpr int kKryThreads = 256;

// jt_i = (3/N_t) Σ_n U_{n,i}² (one thread per point, n in order)
__global__ void __launch_bounds__(256)
k_tavg_jt(const double* __restrict__ U, double* __restrict__ jt, int64_t ns, int nt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int n = 0; n < nt; ++n) {
      const double u = __ldg(U + (size_t)n * ns + i);
      s += u * u;
    }
    jt[i] = 3.0 * s / nt;
  }
}

// block partial sums of x (fixed partition) → part[blockIdx.x]
__global__ void __launch_bounds__(kKryThreads)
k_block_sum(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double sh[kKryThreads / 32];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  double s = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) s += x[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kKryThreads / 32; ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
}

// J̄ = Σ part / ns - c (every block re-sums the partials in the same order), w'_i = jt_i - c - J̄;
// block 0 publishes J̄ to the device stats (the scalar preconditioner's divisor reads it)
__global__ void __launch_bounds__(256)
k_wprime(const double* __restrict__ jt, const double* __restrict__ part, int nparts, int64_t ns, double c,
         double* __restrict__ w, DevStats* st) {
  double t = 0.0;
  for (int b = 0; b < nparts; ++b) t += part[b];
  const double jbar = t / (double)ns - c;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->jbar = jbar;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = jt[i] - c - jbar;
}

// out_n = Δ_h (w ⊙ x_n) on every time slice, 2D Neumann (ghost reflection)
__global__ void __launch_bounds__(256)
k_lap_w(const double* __restrict__ x, const double* __restrict__ w, double* __restrict__ out, int nx, int ny,
        int nt, double inv_h2) {
  const int64_t ns = (int64_t)nx * ny, total = ns * nt;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = k / ns, i = k - n * ns;
    const int iy = (int)(i / nx), ix = (int)(i - (int64_t)iy * nx);
    const double* s = x + n * ns;
    auto q = [&](int xx, int yy) {
      xx = xx < 0 ? -xx : (xx >= nx ? 2 * (nx - 1) - xx : xx);
      yy = yy < 0 ? -yy : (yy >= ny ? 2 * (ny - 1) - yy : yy);
      const int64_t j = (int64_t)yy * nx + xx;
      return __ldg(w + j) * s[j];
    };
    out[k] = (((q(ix - 1, iy) + q(ix + 1, iy)) + (q(ix, iy - 1) + q(ix, iy + 1))) - 4.0 * q(ix, iy)) * inv_h2;
  }
}

// part[i * gridDim.x + b] = Σ_{k ∈ block b} V_i[k] y[k], i < nv (V_i = V + i·ld)
__global__ void __launch_bounds__(kKryThreads)
k_mdot(const double* __restrict__ V, int64_t ld, int nv, const double* __restrict__ y, int64_t n,
       double* __restrict__ part) {
  __shared__ double sh[kKryThreads / 32];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  for (int v = 0; v < nv; ++v) {
    const double* a = V + v * ld;
    double s = 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) s += a[i] * y[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kKryThreads / 32; ++w) t += sh[w];
      part[(int64_t)v * gridDim.x + blockIdx.x] = t;
    }
    __syncthreads();
  }
}

// out[i] = Σ_b part[i * nb + b] (one block per i, fixed-order tree)
__global__ void __launch_bounds__(256)
k_mdot_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double sh[256];
  const double* p = part + (int64_t)blockIdx.x * nb;
  double t = 0.0;
  for (int b = threadIdx.x; b < nb; b += 256) t += p[b];
  sh[threadIdx.x] = t;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}

// y += s · Σ_i coef[i] V_i   (coef on the device)
__global__ void __launch_bounds__(256)
k_maxpy(double* __restrict__ y, const double* __restrict__ V, int64_t ld, int nv, const double* __restrict__ coef,
        double s, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int v = 0; v < nv; ++v) acc += __ldg(coef + v) * V[v * ld + k];
    y[k] += s * acc;
  }
}

// y = a·x + b·y
__global__ void __launch_bounds__(256)
k_axpby(double* __restrict__ y, const double* __restrict__ x, double a, double b, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    y[k] = a * x[k] + b * y[k];
}

__global__ void k_reset_dmax(DevStats* st) { st->dmax_bits = 0ull; }

// ‖x‖∞ → st->dmax_bits (bit-pattern max; NaN sorts above +inf)
__global__ void __launch_bounds__(256)
k_amax_stats(const double* __restrict__ x, int64_t n, DevStats* st) {
  unsigned long long b = 0ull;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    b = max(b, (unsigned long long)__double_as_longlong(x[k]) & 0x7fffffffffffffffull);
  b = warp_max_u64(b);
  if ((threadIdx.x & 31) == 0 && b) atomicMax(&st->dmax_bits, b);
}

// ---------------------------------------------------------------- device-side Arnoldi (graph)
// One GMRES cycle's Arnoldi steps run as the body of a conditional WHILE graph node: the step
// index j, the Hessenberg column, the Givens rotations and the residual estimate live in KryDev on
// the device, every kernel takes j from there, and k_kry_tail decides whether the loop goes on
// (cudaGraphSetConditional) — no host round trip per Krylov step.  The arithmetic (partition and
// order of the dot products, the combination, the rotation formulas) is the host loop's.
constexpr int kKryMaxM = 30;                 // GMRES restart length (kKryM in paradiag.cu)
struct KryDev {
  int j;                                     // next Arnoldi column (basis vectors 0..j exist)
  int steps;                                 // Arnoldi steps taken by the cycle
  double bn, tol;                            // ‖b'‖ and the relative tolerance
  double hn2;                                // ‖v_{j+1}‖² before normalisation
  double a_scale;                            // 1/hn - 1 for the normalising axpby (host loop's form)
  double H[(kKryMaxM + 1) * kKryMaxM];       // row-major (i, j) at i·M + j
  double cs[kKryMaxM], sn[kKryMaxM], g[kKryMaxM + 1];
  double hcol[kKryMaxM + 1];                 // this pass's projections
};

// kin = V_j
__global__ void __launch_bounds__(256)
k_kry_copy_in(const double* __restrict__ V, int64_t n, const KryDev* __restrict__ kd, double* __restrict__ kin) {
  const double* v = V + (int64_t)kd->j * n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    kin[k] = v[k];
}
// V_{j+1} = 1·V_j + (-1)·K V_j  (A v = v - K v, k_axpby's form)
__global__ void __launch_bounds__(256)
k_kry_sub(double* __restrict__ V, int64_t n, const KryDev* __restrict__ kd, const double* __restrict__ kin,
          const double* __restrict__ kout) {
  double* y = V + (int64_t)(kd->j + 1) * n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    y[k] = 1.0 * kin[k] + -1.0 * kout[k];
}
// projections of V_{j+1} on V_0..V_j (NORM: ‖V_{j+1}‖² alone), k_mdot's partition and order
template <bool NORM>
__global__ void __launch_bounds__(kKryThreads)
k_kry_mdot(const double* __restrict__ V, int64_t n, const KryDev* __restrict__ kd, double* __restrict__ part) {
  __shared__ double sh[kKryThreads / 32];
  const int j = kd->j;
  const double* y = V + (int64_t)(j + 1) * n;
  const int nv = NORM ? 1 : j + 1;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  for (int v = 0; v < nv; ++v) {
    const double* a = NORM ? y : V + v * n;
    double s = 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) s += a[i] * y[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kKryThreads / 32; ++w) t += sh[w];
      part[(int64_t)v * gridDim.x + blockIdx.x] = t;
    }
    __syncthreads();
  }
}
// k_mdot_final's tree; NORM: → hn2, else → hcol[i] and H(i, j) += hcol[i]  (blocks i > j idle)
template <bool NORM>
__global__ void __launch_bounds__(256)
k_kry_final(const double* __restrict__ part, int nb, KryDev* __restrict__ kd) {
  __shared__ double sh[256];
  const int j = kd->j;
  if (!NORM && (int)blockIdx.x > j) return;
  const double* p = part + (int64_t)blockIdx.x * nb;
  double t = 0.0;
  for (int b = threadIdx.x; b < nb; b += 256) t += p[b];
  sh[threadIdx.x] = t;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (NORM) {
      kd->hn2 = sh[0];
    } else {
      kd->hcol[blockIdx.x] = sh[0];
      kd->H[blockIdx.x * kKryMaxM + j] += sh[0];
    }
  }
}
// V_{j+1} += -1 · Σ_{i≤j} hcol[i] V_i  (k_maxpy with s = -1)
__global__ void __launch_bounds__(256)
k_kry_maxpy(double* __restrict__ V, int64_t n, const KryDev* __restrict__ kd) {
  const int nv = kd->j + 1;
  double* y = V + (int64_t)nv * n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int v = 0; v < nv; ++v) acc += kd->hcol[v] * V[v * n + k];
    y[k] += -1.0 * acc;
  }
}
// the host loop's step epilogue on one thread: H(j+1, j), previous and new Givens rotations, the
// residual estimate, the stop test; j advances and the WHILE node's condition is set
__global__ void k_kry_tail(KryDev* kd, cudaGraphConditionalHandle cond) {
  const int j = kd->j;
  const double hn = sqrt(kd->hn2);
  double* H = kd->H;
  auto Hij = [&](int i, int c) -> double& { return H[i * kKryMaxM + c]; };
  Hij(j + 1, j) = hn;
  kd->a_scale = hn > 0.0 ? 1.0 / hn - 1.0 : 0.0;
  for (int i = 0; i < j; ++i) {
    const double a = Hij(i, j), c2 = Hij(i + 1, j);
    Hij(i, j) = kd->cs[i] * a + kd->sn[i] * c2;
    Hij(i + 1, j) = -kd->sn[i] * a + kd->cs[i] * c2;
  }
  const double a = Hij(j, j), c2 = Hij(j + 1, j), rr = hypot(a, c2);
  kd->cs[j] = rr > 0.0 ? a / rr : 1.0;
  kd->sn[j] = rr > 0.0 ? c2 / rr : 0.0;
  Hij(j, j) = rr;
  Hij(j + 1, j) = 0.0;
  kd->g[j + 1] = -kd->sn[j] * kd->g[j];
  kd->g[j] = kd->cs[j] * kd->g[j];
  kd->steps += 1;
  const bool stop = fabs(kd->g[j + 1]) <= kd->tol * kd->bn || hn == 0.0;
  kd->j = j + 1;
  cudaGraphSetConditional(cond, (!stop && j + 1 < kKryMaxM) ? 1u : 0u);
}
// V_j (the new column, j already advanced) = a·V_j + 1·V_j, a = 1/hn - 1 (host loop's form)
__global__ void __launch_bounds__(256)
k_kry_scale(double* __restrict__ V, int64_t n, const KryDev* __restrict__ kd) {
  if (kd->a_scale == 0.0 && kd->hn2 == 0.0) return;
  double* y = V + (int64_t)kd->j * n;
  const double a = kd->a_scale;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    y[k] = a * y[k] + 1.0 * y[k];
}

}  // namespace pd
