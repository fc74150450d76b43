// k_tlong.cuh — Steps (1)-(3) along time for long windows (N_t > 4096; SURVEY §8(f) NEXT-3:
// "Δt = 10⁻⁶, i.e. N_t = 10⁶ ... four iterations").
//
// A pencil of N_t = 2^20 complex values (16 MB) does not fit on chip, so the time DFT runs as a
// four-step FFT over HBM: N = N1·N2, n = N2·n1 + n2, k = k1 + N1·k2,
//   X[k1 + N1 k2] = Σ_{n2} W_{N2}^{n2 k2} · W_N^{n2 k1} · Σ_{n1} W_{N1}^{n1 k1} x[N2 n1 + n2].
// Pass A does the length-N1 transforms (stride N2 rows) and the W_N^{n2 k1} twiddle, pass B the
// length-N2 transforms; both are the register-resident warp FFT of fft4.cuh (N1, N2 ≤ 1024).
// Every pass stages a [transform length][8 pencil pairs] tile in shared memory so that HBM is
// touched in 128-byte row segments (8 complex pencils side by side), never pencil by pencil.
//
// Data (all row-major, time slowest):
//   in/out  real    [N][ns]       spatially transformed residual / correction (ns = N_x·N_y modes)
//   Y       complex [N1][N2][P]   after pass A (forward) / before pass A (inverse), P = ⌈ns/2⌉
//   X       complex [N][P]        the spectrum, bin-major; Step (2) divides it in place
// Two real pencils (modes 2p, 2p+1) share one complex pencil z = γ_j (r_j[2p] + i r_j[2p+1]) as in
// k_time.cuh; the divide kernel separates the Hermitian pair from bins k and N−k (both rows of X),
// divides each by its mode's shifted eigenvalue and recombines.
// Inverse: pass B with conjugate roots and W_N^{-n2 k1}, then pass A with conjugate roots and the
// Γ_α⁻¹·(1/N_t)·(spatial normalisation) scale.
#pragma once
#include "common.cuh"
#include "fft4.cuh"
#include "k_time.cuh"

namespace pd {

constexpr int kTlPairs = 8;                  // pencil pairs per CTA = warps per CTA
constexpr int kTlThreads = kTlPairs * 32;
constexpr int kTlRowD = 2 * kTlPairs + 2;    // staged row pitch in doubles (16 + 2 pad: 144 B)
constexpr int kTlRowC = kTlRowD / 2;         // ... in complex slots
constexpr size_t kTlSmem = (size_t)1024 * kTlRowD * sizeof(double);   // 147456 B ≥ 8 × kWarpScratch slots

struct TlongParams {
  int N, log2N;            // N_t
  int N1, N2;              // N = N1·N2, both in [32, 1024]
  int log2N1, log2N2;
  int64_t ns;              // real columns per time row
  int64_t ld;              // row pitch (doubles) of the real in/out arrays: ns, or 2P (even: 16-byte pairs)
  int64_t P;               // complex pencil pairs = ⌈ns/2⌉ (row pitch of Y and X)
  int64_t nch;             // pair chunks = ⌈P/8⌉
  const double2* tw;       // tw[j] = exp(-2πi j / 2^twlog)
  int twlog;
  TimeParams T;            // Step-(2) divisor tables (dl, el, l3, lamx, kind, b2, e2, st, nx, ns)
  // Γ_α split over the four-step index n = N2·n1 + n2: γ_n = ghi[n1]·glo[n2] and
  // scale/γ_n = gihi[n1]·gilo[n2] (one extra rounding; coalesced instead of stride-N2 gathers)
  const double* ghi;
  const double* glo;
  const double* gihi;
  const double* gilo;
  // mixed-radix factors (k_tmix.cuh; N1, N2 products of 2, 4, 5, 8): radix plans, root tables
  // mt1[j] = W_{N1}^j, mt2[j] = W_{N2}^j, mtN[b] = W_N^b (b < N2)
  int mixed;
  int mxp;                 // pencil pairs per CTA of the mixed passes (8 or 4; fused pass B: mxp/2 per group)
  int nst1, nst2;
  int8_t plan1[12], plan2[12];
  const double2* mt1;
  const double2* mt2;
  const double2* mtN;
  // digit reversal of the DIF plans: rev[pos] = frequency at DIF output position, irev its inverse
  const int* rev1;
  const int* rev2;
  const int* irev1;
  const int* irev2;
};

#ifdef PD_TLONG_KERNELS     // defined only in tlong.cu (the engine sees TlongParams alone)
PD_DEV double2 tl_tw(const TlongParams& Q, int e) {
  return __ldg(Q.tw + ((size_t)(e & (Q.N - 1)) << (Q.twlog - Q.log2N)));
}

// The four-step twiddles of one lane: W_N^{±b·(a + E·r)}, r = 0..31, as f·lo[r&7]·hi[r>>3] with
// f = W_N^{±b·a} and lo/hi the TwPow powers of W_N^{±b·E}: 6 table loads instead of 32 gathers.
template <int E, int SIGN>
struct TlTwiddle {
  TwPow<32, SIGN> w;
  PD_DEV TlTwiddle(const TlongParams& Q, int a, int b) : w(b * E, Q.log2N, Q.tw, Q.twlog) {
    double2 f = tl_tw(Q, a * b);
    if (SIGN > 0) f.y = -f.y;
#pragma unroll
    for (int k = 0; k < 8; ++k) w.lo[k] = cmul(w.lo[k], f);
  }
  PD_DEV double2 apply(double2 v, int r) const {
    const double2 a = cmul(v, w.lo[r & 7]);
    return (r >> 3) ? cmul(a, w.hi[r >> 3]) : a;
  }
};

// Pass A forward: rows n = N2·n1 + n2a + g (g < G), columns 16·chunk .. +16 of the real input;
// z = γ_n (r[2p] + i r[2p+1]); length-N1 DFT over n1; × W_N^{n2 k}; store Y[k][n2][p].
template <int E>
__global__ void __launch_bounds__(kTlThreads, 1)
k_tl_a_fwd(const double* __restrict__ in, double2* __restrict__ Y, TlongParams Q) {
  constexpr int G = 32 / E, L = 32 * E;
  extern __shared__ double2 sm[];
  double* sd = reinterpret_cast<double*>(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chunk = blockIdx.x % Q.nch;
  const int n2a = (int)(blockIdx.x / Q.nch) * G;
  const int64_t c0 = chunk * (2 * kTlPairs);
  if (!(Q.ld & 1)) {                                    // even pitch: 16-byte pencil pairs
    for (int idx = threadIdx.x; idx < G * L * kTlPairs; idx += kTlThreads) {
      const int w = idx & 7, row = idx >> 3;
      const int g = row % G, n1 = row / G;
      const int64_t n = (int64_t)Q.N2 * n1 + n2a + g;
      double* d = sd + (g * L + n1) * kTlRowD + 2 * w;
      if (chunk * kTlPairs + w < Q.P) cp_async16(d, in + n * Q.ld + c0 + 2 * w);
      else d[0] = d[1] = 0.0;
    }
  } else {
    for (int idx = threadIdx.x; idx < G * L * 16; idx += kTlThreads) {
      const int c = idx & 15, row = idx >> 4;          // row = n1·G + g: consecutive g are adjacent rows
      const int g = row % G, n1 = row / G;
      const int64_t n = (int64_t)Q.N2 * n1 + n2a + g;
      double* d = sd + (g * L + n1) * kTlRowD + c;
      if (c0 + c < Q.ns) cp_async8(d, in + n * Q.ld + c0 + c);
      else *d = 0.0;
    }
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  double2 v[32];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int n1 = lane + 32 * e;
      const double2 z = *reinterpret_cast<const double2*>(sd + (g * L + n1) * kTlRowD + 2 * warp);
      const double s = __ldg(Q.ghi + n1) * __ldg(Q.glo + n2a + g);
      v[g * E + e] = make_double2(z.x * s, z.y * s);
    }
  __syncthreads();                                      // the FFT scratch overlaps the staged tile
  fft4_s1_to_s2<E, -1>(v, sm + warp * kWarpScratch, Q.log2N1, Q.tw, Q.twlog, lane);
  __syncthreads();
  {
    const int g = lane / E, k1 = lane % E, n2 = n2a + g;
    const TlTwiddle<E, -1> tw(Q, k1, n2);               // W_N^{n2 (k1 + E r)}
#pragma unroll
    for (int r = 0; r < 32; ++r) sm[(g * L + k1 + E * r) * kTlRowC + warp] = tw.apply(v[r], r);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * L * kTlPairs; idx += kTlThreads) {
    const int w = idx & 7, row = idx >> 3;
    const int g = row % G, k = row / G;
    const int64_t p = chunk * kTlPairs + w;
    if (p < Q.P) Y[((int64_t)k * Q.N2 + n2a + g) * Q.P + p] = sm[(g * L + k) * kTlRowC + w];
  }
}

// Pass B forward: Y rows (k1a + g)·N2 + n2; length-N2 DFT over n2; store X[(k1a + g) + N1·k2][p].
template <int E>
__global__ void __launch_bounds__(kTlThreads, 1)
k_tl_b_fwd(const double2* __restrict__ Y, double2* __restrict__ X, TlongParams Q) {
  constexpr int G = 32 / E, L = 32 * E;
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chunk = blockIdx.x % Q.nch;
  const int k1a = (int)(blockIdx.x / Q.nch) * G;
  for (int idx = threadIdx.x; idx < G * L * kTlPairs; idx += kTlThreads) {
    const int w = idx & 7, row = idx >> 3;
    const int n2 = row % L, g = row / L;                // consecutive n2 are adjacent rows of Y
    const int64_t p = chunk * kTlPairs + w;
    double2* d = sm + (g * L + n2) * kTlRowC + w;
    if (p < Q.P) cp_async16(d, Y + ((int64_t)(k1a + g) * Q.N2 + n2) * Q.P + p);
    else *d = make_double2(0.0, 0.0);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  double2 v[32];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < E; ++e) v[g * E + e] = sm[(g * L + lane + 32 * e) * kTlRowC + warp];
  __syncthreads();
  fft4_s1_to_s2<E, -1>(v, sm + warp * kWarpScratch, Q.log2N2, Q.tw, Q.twlog, lane);
  __syncthreads();
  {
    const int g = lane / E, ka = lane % E;
#pragma unroll
    for (int r = 0; r < 32; ++r) sm[(g * L + ka + E * r) * kTlRowC + warp] = v[r];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * L * kTlPairs; idx += kTlThreads) {
    const int w = idx & 7, row = idx >> 3;
    const int g = row % G, k2 = row / G;                // consecutive g are adjacent bins
    const int64_t p = chunk * kTlPairs + w;
    if (p < Q.P) X[((int64_t)(k1a + g) + (int64_t)Q.N1 * k2) * Q.P + p] = sm[(g * L + k2) * kTlRowC + w];
  }
}

// Step (2): separate the packed pair from bins k and N−k, divide each by its mode's shifted
// eigenvalue (d_k + e_k μ_s [+ λ_{3,k} Λ_s]; CH: J̄ from the device stats), recombine in place.
__global__ void __launch_bounds__(256)
k_tl_divide(double2* __restrict__ X, TlongParams Q) {
  const int64_t half = Q.N >> 1, total = (half + 1) * Q.P;
  const double jbar = Q.T.kind >= 2 ? Q.T.st->jbar : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / Q.P, p = i - k * Q.P;
    const int64_t km = k == 0 ? 0 : Q.N - k;          // the Hermitian mirror bin (any N)
    const double2 Zl = X[k * Q.P + p], Zm = X[km * Q.P + p];
    const double2 A = make_double2(0.5 * (Zl.x + Zm.x), 0.5 * (Zl.y - Zm.y));
    const double2 B = make_double2(0.5 * (Zl.y + Zm.y), -0.5 * (Zl.x - Zm.x));
    const int64_t sa = 2 * p, sb = sa + 1;
    const bool hb = sb < Q.ns;
    const double2 d = __ldg(Q.T.dl + k);
    const double mua = mode_mu(sa, Q.T, jbar);
    const double mub = hb ? mode_mu(sb, Q.T, jbar) : mua;
    const double2 fa = cinv_fast(shifted(d, Q.T.el, (int)k, mua, Q.T.l3, Q.T.l3 ? mode_lam(sa, Q.T) : 0.0));
    const double2 fb = cinv_fast(shifted(d, Q.T.el, (int)k, mub, Q.T.l3, Q.T.l3 && hb ? mode_lam(sb, Q.T) : 0.0));
    const double2 Af = cmul(A, fa), Bf = cmul(B, fb);
    X[k * Q.P + p] = make_double2(Af.x - Bf.y, Af.y + Bf.x);
    if (km != k) X[km * Q.P + p] = make_double2(Af.x + Bf.y, Bf.x - Af.y);
  }
}

// Pass B forward + Step (2) + pass B inverse in one kernel, for N2 = 1024 (one k1 per transform
// group): a CTA takes the k1 and N1−k1 groups (k1 = 0 pairs with N1/2, both self-mirrored) for
// 4 pencil pairs, so every bin k = k1 + N1·k2 finds its mirror N−k = (N1−k1) + N1·(N2−1−k2) in
// shared memory.  The forward FFT leaves bin k2 = lane + 32r in register r, which is exactly the
// input layout of the inverse FFT, so the divided spectrum never leaves registers; Y is read and
// written once (in place) instead of three round trips through X.
#ifndef PD_FB_PAIRS
#define PD_FB_PAIRS 2
#endif
constexpr int kFbPairs = PD_FB_PAIRS;                 // pencil pairs per group (2 groups per CTA)
constexpr int kFbThreads = 2 * kFbPairs * 32;
constexpr int kFbRowC = kFbPairs + 1;                 // staged row pitch (complex)
constexpr size_t kFbSmem = (size_t)2 * 1024 * kFbRowC * sizeof(double2);   // 96 KB (2 pairs: two CTAs per SM)

template <bool PLAIN>      // PLAIN: θ = 1 and no λ₃ term, divisor d_k + μ
__global__ void __launch_bounds__(kFbThreads, kFbPairs <= 2 ? 2 : 1)
k_tl_b_fused(double2* __restrict__ Y, TlongParams Q) {
  constexpr int L = 1024;
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nch4 = (Q.P + kFbPairs - 1) / kFbPairs;
  const int64_t chunk = blockIdx.x % nch4;
  const int j = (int)(blockIdx.x / nch4);               // 0: (0, N1/2); j ≥ 1: (j, N1 - j)
  const int k1b = j == 0 ? Q.N1 / 2 : Q.N1 - j;        // the second group's k1
  for (int idx = threadIdx.x; idx < 2 * L * kFbPairs; idx += kFbThreads) {
    const int w = idx % kFbPairs, row = idx / kFbPairs;
    const int n2 = row & (L - 1), grp = row >> 10;
    const int64_t p = chunk * kFbPairs + w;
    double2* d = sm + (grp * L + n2) * kFbRowC + w;
    if (p < Q.P) cp_async16(d, Y + ((int64_t)(grp ? k1b : j) * L + n2) * Q.P + p);
    else *d = make_double2(0.0, 0.0);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  const int grp = warp / kFbPairs, pw = warp % kFbPairs;
  const int k1 = grp ? k1b : j;
  double2 v[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = sm[(grp * L + lane + 32 * e) * kFbRowC + pw];
  __syncthreads();
  fft4_s1_to_s2<32, -1>(v, sm + warp * kWarpScratch, Q.log2N2, Q.tw, Q.twlog, lane);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 32; ++r) sm[(grp * L + lane + 32 * r) * kFbRowC + pw] = v[r];
  __syncthreads();
  {
    // mirror group and bin: k1 = 0 → (same, (N2 - k2) mod N2); k1 = N1/2 → (same, N2-1-k2);
    // otherwise (other group, N2-1-k2)
    const int mg = (j == 0) ? grp : 1 - grp;
    const bool zero = (j == 0 && grp == 0);
    const int64_t p = chunk * kFbPairs + pw;
    const int64_t sa = 2 * p, sb = sa + 1;
    const bool hb = sb < Q.ns;
    const double jbar = Q.T.kind >= 2 ? Q.T.st->jbar : 0.0;
    const double mua = mode_mu(sa, Q.T, jbar);
    const double mub = hb ? mode_mu(sb, Q.T, jbar) : mua;
    const double lama = Q.T.l3 ? mode_lam(sa, Q.T) : 0.0;
    const double lamb = Q.T.l3 && hb ? mode_lam(sb, Q.T) : 0.0;
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int k2 = lane + 32 * r;
      const int k2m = zero ? ((L - k2) & (L - 1)) : (L - 1 - k2);
      const int k = k1 + Q.N1 * k2;
      const double2 Zl = v[r], Zm = sm[(mg * L + k2m) * kFbRowC + pw];
      const double2 A = make_double2(0.5 * (Zl.x + Zm.x), 0.5 * (Zl.y - Zm.y));
      const double2 B = make_double2(0.5 * (Zl.y + Zm.y), -0.5 * (Zl.x - Zm.x));
      const double2 d = __ldg(Q.T.dl + k);
      double2 Af, Bf;
      if (PLAIN) {
        Af = cmul(A, cinv_fast(make_double2(d.x + mua, d.y)));
        Bf = cmul(B, cinv_fast(make_double2(d.x + mub, d.y)));
      } else {
        Af = cmul(A, cinv_fast(shifted(d, Q.T.el, k, mua, Q.T.l3, lama)));
        Bf = cmul(B, cinv_fast(shifted(d, Q.T.el, k, mub, Q.T.l3, lamb)));
      }
      v[r] = make_double2(Af.x - Bf.y, Af.y + Bf.x);
    }
  }
  __syncthreads();                                      // all mirrors read before the scratch reuse
  fft4_s1_to_s2<32, +1>(v, sm + warp * kWarpScratch, Q.log2N2, Q.tw, Q.twlog, lane);
  __syncthreads();
  {
    const TlTwiddle<32, +1> tw(Q, lane, k1);            // W_N^{-k1 n2}, n2 = lane + 32 r
#pragma unroll
    for (int r = 0; r < 32; ++r) sm[(grp * L + lane + 32 * r) * kFbRowC + pw] = tw.apply(v[r], r);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < 2 * L * kFbPairs; idx += kFbThreads) {
    const int w = idx % kFbPairs, row = idx / kFbPairs;
    const int n2 = row & (L - 1), g = row >> 10;
    const int64_t p = chunk * kFbPairs + w;
    if (p < Q.P) Y[((int64_t)(g ? k1b : j) * L + n2) * Q.P + p] = sm[(g * L + n2) * kFbRowC + w];
  }
}

// Pass B inverse: X rows (k1a + g) + N1·k2; length-N2 inverse DFT over k2; × W_N^{-n2 k1};
// store Y[k1][n2][p].
template <int E>
__global__ void __launch_bounds__(kTlThreads, 1)
k_tl_b_inv(const double2* __restrict__ X, double2* __restrict__ Y, TlongParams Q) {
  constexpr int G = 32 / E, L = 32 * E;
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chunk = blockIdx.x % Q.nch;
  const int k1a = (int)(blockIdx.x / Q.nch) * G;
  for (int idx = threadIdx.x; idx < G * L * kTlPairs; idx += kTlThreads) {
    const int w = idx & 7, row = idx >> 3;
    const int g = row % G, k2 = row / G;
    const int64_t p = chunk * kTlPairs + w;
    double2* d = sm + (g * L + k2) * kTlRowC + w;
    if (p < Q.P) cp_async16(d, X + ((int64_t)(k1a + g) + (int64_t)Q.N1 * k2) * Q.P + p);
    else *d = make_double2(0.0, 0.0);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  double2 v[32];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < E; ++e) v[g * E + e] = sm[(g * L + lane + 32 * e) * kTlRowC + warp];
  __syncthreads();
  fft4_s1_to_s2<E, +1>(v, sm + warp * kWarpScratch, Q.log2N2, Q.tw, Q.twlog, lane);
  __syncthreads();
  {
    const int g = lane / E, na = lane % E, k1 = k1a + g;
    const TlTwiddle<E, +1> tw(Q, na, k1);               // W_N^{-k1 (na + E r)}
#pragma unroll
    for (int r = 0; r < 32; ++r) sm[(g * L + na + E * r) * kTlRowC + warp] = tw.apply(v[r], r);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * L * kTlPairs; idx += kTlThreads) {
    const int w = idx & 7, row = idx >> 3;
    const int n2 = row % L, g = row / L;
    const int64_t p = chunk * kTlPairs + w;
    if (p < Q.P) Y[((int64_t)(k1a + g) * Q.N2 + n2) * Q.P + p] = sm[(g * L + n2) * kTlRowC + w];
  }
}

// Pass A inverse: Y rows k1·N2 + n2a + g; length-N1 inverse DFT over k1; × ginv[n] (Γ_α⁻¹ and all
// normalisations); real part → column 2p, imaginary part → 2p+1 of row n = N2·n1 + n2a + g.
template <int E>
__global__ void __launch_bounds__(kTlThreads, 1)
k_tl_a_inv(const double2* __restrict__ Y, double* __restrict__ out, TlongParams Q) {
  constexpr int G = 32 / E, L = 32 * E;
  extern __shared__ double2 sm[];
  double* sd = reinterpret_cast<double*>(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chunk = blockIdx.x % Q.nch;
  const int n2a = (int)(blockIdx.x / Q.nch) * G;
  const int64_t c0 = chunk * (2 * kTlPairs);
  for (int idx = threadIdx.x; idx < G * L * kTlPairs; idx += kTlThreads) {
    const int w = idx & 7, row = idx >> 3;
    const int g = row % G, k1 = row / G;
    const int64_t p = chunk * kTlPairs + w;
    double2* d = sm + (g * L + k1) * kTlRowC + w;
    if (p < Q.P) cp_async16(d, Y + ((int64_t)k1 * Q.N2 + n2a + g) * Q.P + p);
    else *d = make_double2(0.0, 0.0);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  double2 v[32];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < E; ++e) v[g * E + e] = sm[(g * L + lane + 32 * e) * kTlRowC + warp];
  __syncthreads();
  fft4_s1_to_s2<E, +1>(v, sm + warp * kWarpScratch, Q.log2N1, Q.tw, Q.twlog, lane);
  __syncthreads();
  {
    const int g = lane / E, na = lane % E;
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int n1 = na + E * r;
      const double s = __ldg(Q.gihi + n1) * __ldg(Q.gilo + n2a + g);
      *reinterpret_cast<double2*>(sd + (g * L + n1) * kTlRowD + 2 * warp) = make_double2(v[r].x * s, v[r].y * s);
    }
  }
  __syncthreads();
  if (!(Q.ld & 1)) {                                    // even pitch: 16-byte pairs (pad column included)
    for (int idx = threadIdx.x; idx < G * L * kTlPairs; idx += kTlThreads) {
      const int w = idx & 7, row = idx >> 3;
      const int g = row % G, n1 = row / G;
      const int64_t n = (int64_t)Q.N2 * n1 + n2a + g;
      if (chunk * kTlPairs + w < Q.P)
        *reinterpret_cast<double2*>(out + n * Q.ld + c0 + 2 * w) =
            *reinterpret_cast<const double2*>(sd + (g * L + n1) * kTlRowD + 2 * w);
    }
  } else {
    for (int idx = threadIdx.x; idx < G * L * 16; idx += kTlThreads) {
      const int c = idx & 15, row = idx >> 4;
      const int g = row % G, n1 = row / G;
      const int64_t n = (int64_t)Q.N2 * n1 + n2a + g;
      if (c0 + c < Q.ns) out[n * Q.ld + c0 + c] = sd[(g * L + n1) * kTlRowD + c];
    }
  }
}
#endif  // PD_TLONG_KERNELS

}  // namespace pd
