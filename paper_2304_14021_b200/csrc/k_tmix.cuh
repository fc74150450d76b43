// k_tmix.cuh — the long-window time pass for N_t with factors 2 and 5 (the
// paper's "Δt = 10⁻⁶, i.e. N_t = 10⁶" run, P:692-699, 10⁶ = 2⁶·5⁶; also N_t = 10⁴, and
// 40000).  Same four-step decomposition and data layout as k_tlong.cuh (N = N1·N2,
// n = N2·n1 + n2, k = k1 + N1·k2; real in/out [N][ld], Y [N1][N2][P], X [N][P]), but the
// transforms of length N1 and N2 (products of 2, 4, 5, 8 — e.g. 1000 = 8·5·5·5) run as in-place
// mixed-radix Cooley–Tukey in shared memory instead of the power-of-two register FFT:
//   forward  = decimation in frequency (natural order in, digit-reversed order out),
//   inverse  = decimation in time with conjugate roots (digit-reversed in, natural out),
// so a forward/inverse pair needs no reordering pass; the digit reversal is folded into the
// global store (forward) and load (inverse) addresses.  A CTA stages a [L][8 pencil pairs] tile
// (128-byte row segments), warp w owns pencil pair w and sweeps its butterflies stage by stage
// (no block barriers inside the transform).
// Twiddles: W_L^e from a table of the length's own roots; the four-step twiddle W_N^{n2·k1} is
// W_{N1}^{a}·W_N^{b} with n2·k1 mod N = a·N2 + b (two table loads, one extra rounding).
#pragma once
#include "common.cuh"
#include "k_tlong.cuh"

namespace pd {

// Digit reversal (tables built on the host, TlongParams.rev* / irev*): for a DIF plan r0, r1, … of
// length L, frequency k = q0 + r0·q1 + r0·r1·q2 + … sits at position pos = q0·(L/r0) + q1·(L/(r0 r1)) + ….

// small DFTs y_q = Σ_t a_t W_R^{SIGN·t·q}, W_R = e^{-2πi/R} (SIGN = -1 forward, +1 inverse), in place
template <int SIGN>
PD_DEV void dft2(double2* a) {
  const double2 t = a[1];
  a[1] = csub(a[0], t);
  a[0] = cadd(a[0], t);
}
template <int SIGN>
PD_DEV double2 mul_mi(double2 v) {       // v · (SIGN == -1 ? -i : +i)
  return SIGN < 0 ? make_double2(v.y, -v.x) : make_double2(-v.y, v.x);
}
template <int SIGN>
PD_DEV void dft4(double2* a) {
  const double2 s0 = cadd(a[0], a[2]), d0 = csub(a[0], a[2]);
  const double2 s1 = cadd(a[1], a[3]), d1 = mul_mi<SIGN>(csub(a[1], a[3]));
  a[0] = cadd(s0, s1);
  a[2] = csub(s0, s1);
  a[1] = cadd(d0, d1);
  a[3] = csub(d0, d1);
}
template <int SIGN>
PD_DEV void dft5(double2* a) {
  // y_q = a0 + Σ_{t=1..4} a_t W^{tq}; pairs (1,4), (2,3): cos/sin of 2π/5, 4π/5
  constexpr double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
  constexpr double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;
  const double2 p1 = cadd(a[1], a[4]), m1 = csub(a[1], a[4]);
  const double2 p2 = cadd(a[2], a[3]), m2 = csub(a[2], a[3]);
  const double2 r1 = make_double2(a[0].x + c1 * p1.x + c2 * p2.x, a[0].y + c1 * p1.y + c2 * p2.y);
  const double2 r2 = make_double2(a[0].x + c2 * p1.x + c1 * p2.x, a[0].y + c2 * p1.y + c1 * p2.y);
  // i·SIGN·(s·m) terms: W^{t} = cos − i sin (forward), so y_1 = r1 − i(s1 m1 + s2 m2) forward
  const double2 i1 = make_double2(s1 * m1.x + s2 * m2.x, s1 * m1.y + s2 * m2.y);
  const double2 i2 = make_double2(s2 * m1.x - s1 * m2.x, s2 * m1.y - s1 * m2.y);
  const double2 j1 = mul_mi<SIGN>(i1), j2 = mul_mi<SIGN>(i2);
  a[0] = make_double2(a[0].x + p1.x + p2.x, a[0].y + p1.y + p2.y);
  a[1] = cadd(r1, j1);
  a[4] = csub(r1, j1);
  a[2] = cadd(r2, j2);
  a[3] = csub(r2, j2);
}
template <int SIGN>
PD_DEV void dft8(double2* a) {
  constexpr double h = 0.70710678118654752440;
  double2 e[4] = {a[0], a[2], a[4], a[6]}, o[4] = {a[1], a[3], a[5], a[7]};
  dft4<SIGN>(e);
  dft4<SIGN>(o);
  // o_q · W_8^{SIGN·... q}: W_8^1 = (1 − i)/√2 forward
  o[1] = SIGN < 0 ? make_double2((o[1].x + o[1].y) * h, (o[1].y - o[1].x) * h)
                  : make_double2((o[1].x - o[1].y) * h, (o[1].y + o[1].x) * h);
  o[2] = mul_mi<SIGN>(o[2]);
  o[3] = SIGN < 0 ? make_double2((o[3].y - o[3].x) * h, -(o[3].x + o[3].y) * h)
                  : make_double2(-(o[3].x + o[3].y) * h, (o[3].x - o[3].y) * h);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    a[q] = cadd(e[q], o[q]);
    a[q + 4] = csub(e[q], o[q]);
  }
}

template <int R, int SIGN>
PD_DEV void dft_r(double2* a) {
  if constexpr (R == 2) dft2<SIGN>(a);
  else if constexpr (R == 4) dft4<SIGN>(a);
  else if constexpr (R == 5) dft5<SIGN>(a);
  else dft8<SIGN>(a);
}

// W_L^{SIGN·e} from tab[j] = e^{-2πi j/L}, 0 <= e < L (a stage's j·q·(L/len) < L since j < len/R, q < R)
template <int SIGN>
PD_DEV double2 mix_root(const double2* __restrict__ tab, int e) {
  double2 w = __ldg(tab + e);
  if (SIGN > 0) w.y = -w.y;
  return w;
}

// One stage of radix R on the pencil x[i·pitch] (i < L) of the calling warp.  Forward (DIF): span
// len → m = len/R: gather a_t = x[b + j + t m], y = DFT_R(a), y_q ·= W_len^{j q}, store at b + j + q m.
// Inverse (DIT, SIGN = +1): span m → len = m R: a_q = x[b + j + q m]·W_len^{-j q}, y = DFT_R^{+}(a),
// store y_t at b + j + t m.  tab = roots of L (W_len^{jq} = W_L^{jq·L/len}).
template <int R, int SIGN>
PD_DEV void mix_stage(double2* x, int pitch, int L, int len, const double2* __restrict__ tab, int lane) {
  const int m = len / R, nb = L / len, stride = L / len;
  for (int idx = lane; idx < nb * m; idx += 32) {
    const int b = (idx / m) * len, j = idx - (idx / m) * m;
    double2 a[R];
#pragma unroll
    for (int t = 0; t < R; ++t) a[t] = x[(b + j + t * m) * pitch];
    if (SIGN > 0) {                                  // DIT: undo the twiddles first
#pragma unroll
      for (int q = 1; q < R; ++q) a[q] = cmul(a[q], mix_root<+1>(tab, j * q * stride));
    }
    dft_r<R, SIGN>(a);
    if (SIGN < 0) {
#pragma unroll
      for (int q = 1; q < R; ++q) a[q] = cmul(a[q], mix_root<-1>(tab, j * q * stride));
    }
#pragma unroll
    for (int t = 0; t < R; ++t) x[(b + j + t * m) * pitch] = a[t];
  }
  __syncwarp();
}

template <int SIGN>
PD_DEV void mix_stage_rt(int R, double2* x, int pitch, int L, int len, const double2* tab, int lane) {
  switch (R) {
    case 2: mix_stage<2, SIGN>(x, pitch, L, len, tab, lane); break;
    case 4: mix_stage<4, SIGN>(x, pitch, L, len, tab, lane); break;
    case 5: mix_stage<5, SIGN>(x, pitch, L, len, tab, lane); break;
    default: mix_stage<8, SIGN>(x, pitch, L, len, tab, lane); break;
  }
}

// Forward (DIF) transform of length L of the warp's pencil: natural in, digit-reversed out
PD_DEV void mix_fft_fwd(double2* x, int pitch, int L, const int8_t* r, int ns, const double2* tab, int lane) {
  int len = L;
  for (int s = 0; s < ns; ++s) {
    mix_stage_rt<-1>(r[s], x, pitch, L, len, tab, lane);
    len /= r[s];
  }
}
// Inverse (DIT, conjugate roots, unnormalised): digit-reversed in, natural out
PD_DEV void mix_fft_inv(double2* x, int pitch, int L, const int8_t* r, int ns, const double2* tab, int lane) {
  int len = 1;
  for (int s = ns - 1; s >= 0; --s) {
    len *= r[s];
    mix_stage_rt<+1>(r[s], x, pitch, L, len, tab, lane);
  }
}

// four-step twiddle W_N^{SIGN·n2·k1} = W_{N1}^{a}·W_N^{b}, n2·k1 mod N = a·N2 + b
template <int SIGN>
PD_DEV double2 mix_tw4(const TlongParams& Q, int n2, int k1) {
  const int e = (n2 * k1) % Q.N, a = e / Q.N2, b = e - a * Q.N2;       // n2·k1 < N ≤ 2^20: 32-bit
  return cmul(mix_root<SIGN>(Q.mt1, a), mix_root<SIGN>(Q.mtN, b));      // mtN[b] = W_N^b, b < N2
}

constexpr int kMxRowC = kTlPairs + 1;                 // staged row pitch (complex): 8 pairs + 1 pad

// Pass A forward: rows n = N2·n1 + n2, 16 real columns (8 pairs) of chunk; z = γ_n (r[2p] + i r[2p+1]);
// length-N1 DFT over n1 (DIF); × W_N^{n2 k1}; store Y[k1][n2][p] (k1 un-reversed).
__global__ void __launch_bounds__(kTlThreads, 1) k_mx_a_fwd(const double* __restrict__ in, double2* __restrict__ Y,
                                                              TlongParams Q) {
  extern __shared__ double2 sm[];
  double* sd = reinterpret_cast<double*>(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chunk = blockIdx.x % Q.nch;
  const int n2 = (int)(blockIdx.x / Q.nch);
  const int64_t c0 = chunk * (2 * kTlPairs);
  const int L = Q.N1;
  for (int idx = threadIdx.x; idx < L * 16; idx += kTlThreads) {      // rows of 16 doubles (128 B)
    const int c = idx & 15, n1 = idx >> 4;
    const int64_t n = (int64_t)Q.N2 * n1 + n2;
    double* d = sd + n1 * 2 * kMxRowC + c;
    if (c0 + c < Q.ns) cp_async8(d, in + n * Q.ld + c0 + c);
    else *d = 0.0;
  }
  cp_async_commit();
  cp_async_wait_all();
  const double g2 = __ldg(Q.glo + n2);
  for (int idx = threadIdx.x; idx < L * 16; idx += kTlThreads) {      // γ_n = ghi[n1]·glo[n2], own elements
    const int c = idx & 15, n1 = idx >> 4;
    sd[n1 * 2 * kMxRowC + c] *= __ldg(Q.ghi + n1) * g2;
  }
  __syncthreads();
  mix_fft_fwd(sm + warp, kMxRowC, L, Q.plan1, Q.nst1, Q.mt1, lane);
  __syncthreads();
  for (int idx = threadIdx.x; idx < L * kTlPairs; idx += kTlThreads) {
    const int w = idx & 7, pos = idx >> 3;
    const int64_t p = chunk * kTlPairs + w;
    const int k1 = __ldg(Q.rev1 + pos);
    if (p < Q.P) Y[((int64_t)k1 * Q.N2 + n2) * Q.P + p] = cmul(sm[pos * kMxRowC + w], mix_tw4<-1>(Q, n2, k1));
  }
}

// Pass B forward: Y rows k1·N2 + n2 (n2 < N2); length-N2 DFT over n2 (DIF); X[k1 + N1·k2][p].
__global__ void __launch_bounds__(kTlThreads, 1) k_mx_b_fwd(const double2* __restrict__ Y, double2* __restrict__ X,
                                                              TlongParams Q) {
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chunk = blockIdx.x % Q.nch;
  const int k1 = (int)(blockIdx.x / Q.nch);
  const int L = Q.N2;
  for (int idx = threadIdx.x; idx < L * kTlPairs; idx += kTlThreads) {
    const int w = idx & 7, n2 = idx >> 3;
    const int64_t p = chunk * kTlPairs + w;
    if (p < Q.P) cp_async16(sm + n2 * kMxRowC + w, Y + ((int64_t)k1 * Q.N2 + n2) * Q.P + p);
    else sm[n2 * kMxRowC + w] = make_double2(0.0, 0.0);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  mix_fft_fwd(sm + warp, kMxRowC, L, Q.plan2, Q.nst2, Q.mt2, lane);
  __syncthreads();
  for (int idx = threadIdx.x; idx < L * kTlPairs; idx += kTlThreads) {
    const int w = idx & 7, pos = idx >> 3;
    const int64_t p = chunk * kTlPairs + w;
    const int k2 = __ldg(Q.rev2 + pos);
    if (p < Q.P) X[((int64_t)k1 + (int64_t)Q.N1 * k2) * Q.P + p] = sm[pos * kMxRowC + w];
  }
}

// Pass B inverse: X[k1 + N1·k2] placed at the digit-reversed position of k2, inverse DIT over k2
// → natural n2; Y[k1][n2].
__global__ void __launch_bounds__(kTlThreads, 1) k_mx_b_inv(const double2* __restrict__ X, double2* __restrict__ Y,
                                                              TlongParams Q) {
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chunk = blockIdx.x % Q.nch;
  const int k1 = (int)(blockIdx.x / Q.nch);
  const int L = Q.N2;
  for (int idx = threadIdx.x; idx < L * kTlPairs; idx += kTlThreads) {
    const int w = idx & 7, k2 = idx >> 3;
    const int64_t p = chunk * kTlPairs + w;
    double2* d = sm + __ldg(Q.irev2 + k2) * kMxRowC + w;
    if (p < Q.P) cp_async16(d, X + ((int64_t)k1 + (int64_t)Q.N1 * k2) * Q.P + p);
    else *d = make_double2(0.0, 0.0);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  mix_fft_inv(sm + warp, kMxRowC, L, Q.plan2, Q.nst2, Q.mt2, lane);
  __syncthreads();
  for (int idx = threadIdx.x; idx < L * kTlPairs; idx += kTlThreads) {
    const int w = idx & 7, n2 = idx >> 3;
    const int64_t p = chunk * kTlPairs + w;
    if (p < Q.P) Y[((int64_t)k1 * Q.N2 + n2) * Q.P + p] = sm[n2 * kMxRowC + w];
  }
}

// Pass A inverse: Y[k1][n2] × W_N^{-n2 k1} at the digit-reversed position of k1, inverse DIT over
// k1 → natural n1; out rows n = N2·n1 + n2 with Γ_α⁻¹·(1/N_t)·(spatial normalisation).
__global__ void __launch_bounds__(kTlThreads, 1) k_mx_a_inv(const double2* __restrict__ Y, double* __restrict__ out,
                                                              TlongParams Q) {
  extern __shared__ double2 sm[];
  double* sd = reinterpret_cast<double*>(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chunk = blockIdx.x % Q.nch;
  const int n2 = (int)(blockIdx.x / Q.nch);
  const int64_t c0 = chunk * (2 * kTlPairs);
  const int L = Q.N1;
  for (int idx = threadIdx.x; idx < L * kTlPairs; idx += kTlThreads) {
    const int w = idx & 7, k1 = idx >> 3;
    const int64_t p = chunk * kTlPairs + w;
    double2* d = sm + __ldg(Q.irev1 + k1) * kMxRowC + w;
    if (p < Q.P) cp_async16(d, Y + ((int64_t)k1 * Q.N2 + n2) * Q.P + p);
    else *d = make_double2(0.0, 0.0);
  }
  cp_async_commit();
  cp_async_wait_all();
  for (int idx = threadIdx.x; idx < L * kTlPairs; idx += kTlThreads) {   // × W_N^{-n2 k1}, own elements
    const int w = idx & 7, k1 = idx >> 3;
    double2* d = sm + __ldg(Q.irev1 + k1) * kMxRowC + w;
    *d = cmul(*d, mix_tw4<+1>(Q, n2, k1));
  }
  __syncthreads();
  mix_fft_inv(sm + warp, kMxRowC, L, Q.plan1, Q.nst1, Q.mt1, lane);
  __syncthreads();
  for (int idx = threadIdx.x; idx < L * 16; idx += kTlThreads) {
    const int c = idx & 15, n1 = idx >> 4;
    const int64_t n = (int64_t)Q.N2 * n1 + n2;
    if (c0 + c < Q.ns)
      out[n * Q.ld + c0 + c] = sd[n1 * 2 * kMxRowC + c] * (__ldg(Q.gihi + n1) * __ldg(Q.gilo + n2));
  }
}

}  // namespace pd
