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

// One stage of radix R on the pencil x[i·pitch] (i < L) of the calling warp group (WPP warps per
// pencil pair, `sub` = the warp's index in its group, group barrier `gbar` between stages).
// Forward (DIF): span len → m = len/R: gather a_t = x[b + j + t m], y = DFT_R(a), y_q ·= W_len^{j q},
// store at b + j + q m.  Inverse (DIT, SIGN = +1): span m → len = m R: a_q = x[b + j + q m]·W_len^{-j q},
// y = DFT_R^{+}(a), store y_t at b + j + t m.  tab = roots of L (W_len^{jq} = W_L^{jq·L/len}).
// idx / m by a 2^20-scaled reciprocal: exact for idx < L/R ≤ 512 and m < 1024 (the error
// idx·(⌈2^20/m⌉ − 2^20/m)/2^20 < 2^-11 stays below the 1/m gap to the next integer).
constexpr int kMxWpp = 2;                                   // warps per pencil pair

PD_DEV void mx_group_sync(int gid) {                        // the kMxWpp warps of pencil group gid
  if (kMxWpp == 1) __syncwarp();
  else asm volatile("bar.sync %0, %1;" ::"r"(gid + 1), "r"(kMxWpp * 32) : "memory");
}

template <int R, int SIGN>
PD_DEV void mix_stage(double2* x, int pitch, int L, int len, const double2* __restrict__ tab, int t0) {
  const int m = len / R, nb = L / len, stride = L / len;
  const unsigned inv_m = ((1u << 20) + (unsigned)m - 1u) / (unsigned)m;
  for (int idx = t0; idx < nb * m; idx += 32 * kMxWpp) {
    const int bq = (int)(((unsigned)idx * inv_m) >> 20);
    const int b = bq * len, j = idx - bq * m;
    double2 a[R];
#pragma unroll
    for (int t = 0; t < R; ++t) a[t] = x[(b + j + t * m) * pitch];
    double2 w[R];                                    // W^{jq}: one load, powers by products (mix_stage_ct)
    w[1] = mix_root<SIGN>(tab, j * stride);
#pragma unroll
    for (int q = 2; q < R; ++q) w[q] = cmul(w[q - 1], w[1]);
    if (SIGN > 0) {                                  // DIT: undo the twiddles first
#pragma unroll
      for (int q = 1; q < R; ++q) a[q] = cmul(a[q], w[q]);
    }
    dft_r<R, SIGN>(a);
    if (SIGN < 0) {
#pragma unroll
      for (int q = 1; q < R; ++q) a[q] = cmul(a[q], w[q]);
    }
#pragma unroll
    for (int t = 0; t < R; ++t) x[(b + j + t * m) * pitch] = a[t];
  }
}

template <int SIGN>
PD_DEV void mix_stage_rt(int R, double2* x, int pitch, int L, int len, const double2* tab, int t0, int gid) {
  switch (R) {
    case 2: mix_stage<2, SIGN>(x, pitch, L, len, tab, t0); break;
    case 4: mix_stage<4, SIGN>(x, pitch, L, len, tab, t0); break;
    case 5: mix_stage<5, SIGN>(x, pitch, L, len, tab, t0); break;
    default: mix_stage<8, SIGN>(x, pitch, L, len, tab, t0); break;
  }
  mx_group_sync(gid);
}

// Compile-time plans (the production lengths: N_t = 10⁶ → L = 1000 = 8·5·5·5, N_t = 10⁴ → L = 100
// = 4·5·5): the same stages with L, the span and the radix as constants, so the index arithmetic
// folds (ncu c6n: integer multiply-adds were the largest instruction class of the runtime-plan
// stages, and their three runtime divisions per stage showed up as I2F stalls) and the butterfly
// loop unrolls.  Identical arithmetic to mix_stage.
template <int R, int L, int LEN, int SIGN, int NTP>
PD_DEV void mix_stage_ct(double2* x, int pitch, const double2* __restrict__ tab, int t0) {
  constexpr int m = LEN / R, nb = L / LEN, stride = L / LEN, cnt = nb * m, IT = (cnt + NTP - 1) / NTP;
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int idx = t0 + it * NTP;
    if (idx < cnt) {
      const int bq = idx / m;
      const int b = bq * LEN, j = idx - bq * m;
      double2 a[R];
#pragma unroll
      for (int t = 0; t < R; ++t) a[t] = x[(b + j + t * m) * pitch];
      // W^{jq} for q = 1..R-1: one table load, the powers by complex products (q - 1 extra roundings;
      // the table gathers were the stage loop's long-scoreboard stalls)
      double2 w[R];
      if (m > 1) {
        w[1] = mix_root<SIGN>(tab, j * stride);
#pragma unroll
        for (int q = 2; q < R; ++q) w[q] = cmul(w[q - 1], w[1]);
      }
      if (SIGN > 0 && m > 1) {
#pragma unroll
        for (int q = 1; q < R; ++q) a[q] = cmul(a[q], w[q]);
      }
      dft_r<R, SIGN>(a);
      if (SIGN < 0 && m > 1) {
#pragma unroll
        for (int q = 1; q < R; ++q) a[q] = cmul(a[q], w[q]);
      }
#pragma unroll
      for (int t = 0; t < R; ++t) x[(b + j + t * m) * pitch] = a[t];
    }
  }
}
template <int L, int LEN, int NTP, int R, int... Rest>
PD_DEV void mix_fwd_ct(double2* x, int pitch, const double2* tab, int t0, int gid) {
  mix_stage_ct<R, L, LEN, -1, NTP>(x, pitch, tab, t0);
  mx_group_sync(gid);
  if constexpr (sizeof...(Rest) > 0) mix_fwd_ct<L, LEN / R, NTP, Rest...>(x, pitch, tab, t0, gid);
}
template <int L, int LEN, int NTP, int R, int... Rest>
PD_DEV void mix_inv_ct(double2* x, int pitch, const double2* tab, int t0, int gid) {
  if constexpr (sizeof...(Rest) > 0) mix_inv_ct<L, LEN / R, NTP, Rest...>(x, pitch, tab, t0, gid);
  mix_stage_ct<R, L, LEN, +1, NTP>(x, pitch, tab, t0);
  mx_group_sync(gid);
}
PD_DEV bool plan_is(const int8_t* r, int ns, int n, int a, int b, int c, int d) {
  return ns == n && r[0] == a && r[1] == b && (n < 3 || r[2] == c) && (n < 4 || r[3] == d);
}

// Forward (DIF) transform of length L of the group's pencil: natural in, digit-reversed out.
// t0 = sub·32 + lane; gid = pencil group (every warp of the group calls, so the barriers match).
PD_DEV void mix_fft_fwd(double2* x, int pitch, int L, const int8_t* r, int ns, const double2* tab, int t0, int gid) {
  constexpr int NTP = kMxWpp * 32;
  if (L == 1000 && plan_is(r, ns, 4, 8, 5, 5, 5)) return mix_fwd_ct<1000, 1000, NTP, 8, 5, 5, 5>(x, pitch, tab, t0, gid);
  if (L == 100 && plan_is(r, ns, 3, 4, 5, 5, 0)) return mix_fwd_ct<100, 100, NTP, 4, 5, 5>(x, pitch, tab, t0, gid);
  int len = L;
  for (int s = 0; s < ns; ++s) {
    mix_stage_rt<-1>(r[s], x, pitch, L, len, tab, t0, gid);
    len /= r[s];
  }
}
// Inverse (DIT, conjugate roots, unnormalised): digit-reversed in, natural out
PD_DEV void mix_fft_inv(double2* x, int pitch, int L, const int8_t* r, int ns, const double2* tab, int t0, int gid) {
  constexpr int NTP = kMxWpp * 32;
  if (L == 1000 && plan_is(r, ns, 4, 8, 5, 5, 5)) return mix_inv_ct<1000, 1000, NTP, 8, 5, 5, 5>(x, pitch, tab, t0, gid);
  if (L == 100 && plan_is(r, ns, 3, 4, 5, 5, 0)) return mix_inv_ct<100, 100, NTP, 4, 5, 5>(x, pitch, tab, t0, gid);
  int len = 1;
  for (int s = ns - 1; s >= 0; --s) {
    len *= r[s];
    mix_stage_rt<+1>(r[s], x, pitch, L, len, tab, t0, gid);
  }
}

// four-step twiddle W_N^{SIGN·n2·k1} = W_{N1}^{a}·W_N^{b}, n2·k1 = a·N2 + b (n2 < N2, k1 < N1, so
// n2·k1 < N: no reduction mod N); a = ⌊e/N2⌋ by the reciprocal inv_n2 = ⌈2^32/N2⌉, exact for
// e < 2^32/N2 (e < N ≤ 2^20, N2 ≤ 1024)
template <int SIGN>
PD_DEV double2 mix_tw4(const TlongParams& Q, int n2, int k1, unsigned inv_n2) {
  const unsigned e = (unsigned)(n2 * k1), a = __umulhi(e, inv_n2), b = e - a * (unsigned)Q.N2;
  return cmul(mix_root<SIGN>(Q.mt1, (int)a), mix_root<SIGN>(Q.mtN, (int)b));      // mtN[b] = W_N^b, b < N2
}
PD_DEV unsigned mx_inv_n2(int N2) { return (unsigned)((0x100000000ull + (unsigned)N2 - 1) / (unsigned)N2); }

// Pass kernels: NP pencil pairs per CTA (8: 128-byte row segments, one CTA per SM; 4: 64-byte
// segments, two CTAs per SM so that one CTA's loads and stores overlap the other's transform).
// Dynamic shared memory: the staged tile [L][NP + 1] complex (sized for L = 1024), then the
// per-CTA tables of the pass: the digit-reversal map of its length (int [1024]) and, for pass A,
// the four-step twiddles of its n2 (complex [1024]).  ncu c6n: the per-element global lookups of
// those tables inside the load / store loops (each behind the previous cp.async or store) were
// the largest long-scoreboard stall; the tables are now built once per CTA, while the tile loads
// are in flight where possible.
template <int NP>
__host__ __device__ constexpr size_t mx_tile_bytes() { return (size_t)1024 * (NP + 1) * sizeof(double2); }
template <int NP>
__host__ __device__ constexpr size_t mx_pass_smem() { return mx_tile_bytes<NP>() + 1024 * sizeof(int) + 1024 * sizeof(double2); }

// Pass A forward: rows n = N2·n1 + n2, 2·NP real columns (NP pairs) of chunk; z = γ_n (r[2p] + i r[2p+1]);
// length-N1 DFT over n1 (DIF); × W_N^{n2 k1}; store Y[k1][n2][p] (k1 un-reversed).
// Two warps per pencil pair (stages split between them, group barriers); pencil pairs past P
// (the padded last chunk) skip the transform.  Rows are staged with 16-byte copies when the row
// pitch is even.
template <int NP>
__global__ void __launch_bounds__(NP * kMxWpp * 32, NP <= 4 ? 2 : 1) k_mx_a_fwd(const double* __restrict__ in, double2* __restrict__ Y,
                                                              TlongParams Q) {
  constexpr int kMxRowC = NP + 1, NT = NP * kMxWpp * 32;   // staged row pitch (complex), threads
  const int64_t nch = (Q.P + NP - 1) / NP;
  extern __shared__ double2 sm[];
  double* sd = reinterpret_cast<double*>(sm);
  int* k1s = reinterpret_cast<int*>(reinterpret_cast<char*>(sm) + mx_tile_bytes<NP>());
  double2* tws = reinterpret_cast<double2*>(k1s + 1024);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pen = warp / kMxWpp, t0 = (warp % kMxWpp) * 32 + lane;
  const int64_t chunk = blockIdx.x % nch;
  const int n2 = (int)(blockIdx.x / nch);
  const int64_t c0 = chunk * (2 * NP);
  const int L = Q.N1;
  const bool v16 = (Q.ld & 1) == 0;
  for (int idx = threadIdx.x; idx < L * NP; idx += NT) {      // column pairs of the staged rows
    const int c = 2 * (idx % NP), n1 = idx / NP;
    const int64_t n = (int64_t)Q.N2 * n1 + n2;
    double* d = sd + n1 * 2 * kMxRowC + c;
    const double* g = in + n * Q.ld + c0 + c;
    if (c0 + c + 1 < Q.ns) {
      if (v16) cp_async16(d, g);
      else { cp_async8(d, g); cp_async8(d + 1, g + 1); }
    } else if (c0 + c < Q.ns) {
      cp_async8(d, g);
      d[1] = 0.0;
    } else {
      d[0] = 0.0;
      d[1] = 0.0;
    }
  }
  cp_async_commit();
  {                                                     // tables while the tile loads are in flight
    const unsigned inv_n2 = mx_inv_n2(Q.N2);
#pragma unroll 4
    for (int pos = threadIdx.x; pos < L; pos += NT) {
      const int k1 = __ldg(Q.rev1 + pos);
      k1s[pos] = k1;
      tws[pos] = mix_tw4<-1>(Q, n2, k1, inv_n2);
    }
  }
  cp_async_wait_all();
  const double g2 = __ldg(Q.glo + n2);
  for (int idx = threadIdx.x; idx < L * NP; idx += NT) {    // γ_n = ghi[n1]·glo[n2], own elements
    const int c = 2 * (idx % NP), n1 = idx / NP;
    const double gm = __ldg(Q.ghi + n1) * g2;
    double* d = sd + n1 * 2 * kMxRowC + c;
    d[0] *= gm;
    d[1] *= gm;
  }
  __syncthreads();
  if (chunk * NP + pen < Q.P) mix_fft_fwd(sm + pen, kMxRowC, L, Q.plan1, Q.nst1, Q.mt1, t0, pen);
  __syncthreads();
  for (int idx = threadIdx.x; idx < L * NP; idx += NT) {
    const int w = idx % NP, pos = idx / NP;
    const int64_t p = chunk * NP + w;
    if (p < Q.P) Y[((int64_t)k1s[pos] * Q.N2 + n2) * Q.P + p] = cmul(sm[pos * kMxRowC + w], tws[pos]);
  }
}

// Pass B forward: Y rows k1·N2 + n2 (n2 < N2); length-N2 DFT over n2 (DIF); X[k1 + N1·k2][p].
template <int NP>
__global__ void __launch_bounds__(NP * kMxWpp * 32, NP <= 4 ? 2 : 1) k_mx_b_fwd(const double2* __restrict__ Y, double2* __restrict__ X,
                                                              TlongParams Q) {
  constexpr int kMxRowC = NP + 1, NT = NP * kMxWpp * 32;
  const int64_t nch = (Q.P + NP - 1) / NP;
  extern __shared__ double2 sm[];
  int* k2s = reinterpret_cast<int*>(reinterpret_cast<char*>(sm) + mx_tile_bytes<NP>());
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pen = warp / kMxWpp, t0 = (warp % kMxWpp) * 32 + lane;
  const int64_t chunk = blockIdx.x % nch;
  const int k1 = (int)(blockIdx.x / nch);
  const int L = Q.N2;
  for (int idx = threadIdx.x; idx < L * NP; idx += NT) {
    const int w = idx % NP, n2 = idx / NP;
    const int64_t p = chunk * NP + w;
    if (p < Q.P) cp_async16(sm + n2 * kMxRowC + w, Y + ((int64_t)k1 * Q.N2 + n2) * Q.P + p);
    else sm[n2 * kMxRowC + w] = make_double2(0.0, 0.0);
  }
  cp_async_commit();
#pragma unroll 4
  for (int pos = threadIdx.x; pos < L; pos += NT) k2s[pos] = __ldg(Q.rev2 + pos);
  cp_async_wait_all();
  __syncthreads();
  if (chunk * NP + pen < Q.P) mix_fft_fwd(sm + pen, kMxRowC, L, Q.plan2, Q.nst2, Q.mt2, t0, pen);
  __syncthreads();
  for (int idx = threadIdx.x; idx < L * NP; idx += NT) {
    const int w = idx % NP, pos = idx / NP;
    const int64_t p = chunk * NP + w;
    if (p < Q.P) X[((int64_t)k1 + (int64_t)Q.N1 * k2s[pos]) * Q.P + p] = sm[pos * kMxRowC + w];
  }
}

// Pass B inverse: X[k1 + N1·k2] placed at the digit-reversed position of k2, inverse DIT over k2
// → natural n2; Y[k1][n2].
template <int NP>
__global__ void __launch_bounds__(NP * kMxWpp * 32, NP <= 4 ? 2 : 1) k_mx_b_inv(const double2* __restrict__ X, double2* __restrict__ Y,
                                                              TlongParams Q) {
  constexpr int kMxRowC = NP + 1, NT = NP * kMxWpp * 32;
  const int64_t nch = (Q.P + NP - 1) / NP;
  extern __shared__ double2 sm[];
  int* ps = reinterpret_cast<int*>(reinterpret_cast<char*>(sm) + mx_tile_bytes<NP>());
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pen = warp / kMxWpp, t0 = (warp % kMxWpp) * 32 + lane;
  const int64_t chunk = blockIdx.x % nch;
  const int k1 = (int)(blockIdx.x / nch);
  const int L = Q.N2;
#pragma unroll 4
  for (int k2 = threadIdx.x; k2 < L; k2 += NT) ps[k2] = __ldg(Q.irev2 + k2);
  __syncthreads();
  for (int idx = threadIdx.x; idx < L * NP; idx += NT) {
    const int w = idx % NP, k2 = idx / NP;
    const int64_t p = chunk * NP + w;
    double2* d = sm + ps[k2] * kMxRowC + w;
    if (p < Q.P) cp_async16(d, X + ((int64_t)k1 + (int64_t)Q.N1 * k2) * Q.P + p);
    else *d = make_double2(0.0, 0.0);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  if (chunk * NP + pen < Q.P) mix_fft_inv(sm + pen, kMxRowC, L, Q.plan2, Q.nst2, Q.mt2, t0, pen);
  __syncthreads();
  for (int idx = threadIdx.x; idx < L * NP; idx += NT) {
    const int w = idx % NP, n2 = idx / NP;
    const int64_t p = chunk * NP + w;
    if (p < Q.P) Y[((int64_t)k1 * Q.N2 + n2) * Q.P + p] = sm[n2 * kMxRowC + w];
  }
}

// Pass A inverse: Y[k1][n2] × W_N^{-n2 k1} at the digit-reversed position of k1, inverse DIT over
// k1 → natural n1; out rows n = N2·n1 + n2 with Γ_α⁻¹·(1/N_t)·(spatial normalisation).
template <int NP>
__global__ void __launch_bounds__(NP * kMxWpp * 32, NP <= 4 ? 2 : 1) k_mx_a_inv(const double2* __restrict__ Y, double* __restrict__ out,
                                                              TlongParams Q) {
  constexpr int kMxRowC = NP + 1, NT = NP * kMxWpp * 32;
  const int64_t nch = (Q.P + NP - 1) / NP;
  extern __shared__ double2 sm[];
  double* sd = reinterpret_cast<double*>(sm);
  int* ps = reinterpret_cast<int*>(reinterpret_cast<char*>(sm) + mx_tile_bytes<NP>());
  double2* tws = reinterpret_cast<double2*>(ps + 1024);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pen = warp / kMxWpp, t0 = (warp % kMxWpp) * 32 + lane;
  const int64_t chunk = blockIdx.x % nch;
  const int n2 = (int)(blockIdx.x / nch);
  const int64_t c0 = chunk * (2 * NP);
  const int L = Q.N1;
  {
    const unsigned inv_n2 = mx_inv_n2(Q.N2);
#pragma unroll 4
    for (int k1 = threadIdx.x; k1 < L; k1 += NT) {
      ps[k1] = __ldg(Q.irev1 + k1);
      tws[k1] = mix_tw4<+1>(Q, n2, k1, inv_n2);
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < L * NP; idx += NT) {
    const int w = idx % NP, k1 = idx / NP;
    const int64_t p = chunk * NP + w;
    double2* d = sm + ps[k1] * kMxRowC + w;
    if (p < Q.P) cp_async16(d, Y + ((int64_t)k1 * Q.N2 + n2) * Q.P + p);
    else *d = make_double2(0.0, 0.0);
  }
  cp_async_commit();
  cp_async_wait_all();
  for (int idx = threadIdx.x; idx < L * NP; idx += NT) {   // × W_N^{-n2 k1}, own elements
    const int w = idx % NP, k1 = idx / NP;
    double2* d = sm + ps[k1] * kMxRowC + w;
    *d = cmul(*d, tws[k1]);
  }
  __syncthreads();
  if (chunk * NP + pen < Q.P) mix_fft_inv(sm + pen, kMxRowC, L, Q.plan1, Q.nst1, Q.mt1, t0, pen);
  __syncthreads();
  const bool v16 = (Q.ld & 1) == 0;
  const double g2 = __ldg(Q.gilo + n2);
  for (int idx = threadIdx.x; idx < L * NP; idx += NT) {
    const int c = 2 * (idx % NP), n1 = idx / NP;
    const int64_t n = (int64_t)Q.N2 * n1 + n2;
    const double gm = __ldg(Q.gihi + n1) * g2;
    const double* d = sd + n1 * 2 * kMxRowC + c;
    double* o = out + n * Q.ld + c0 + c;
    if (c0 + c + 1 < Q.ns) {
      if (v16) *reinterpret_cast<double2*>(o) = make_double2(d[0] * gm, d[1] * gm);
      else { o[0] = d[0] * gm; o[1] = d[1] * gm; }
    } else if (c0 + c < Q.ns) {
      o[0] = d[0] * gm;
    }
  }
}

// Pass B forward + Step (2) + pass B inverse in one kernel for the mixed-radix split (the
// counterpart of k_tl_b_fused): a CTA holds the k1 = j and k1 = N1 − j groups (j = 0 pairs with
// N1/2 when N1 is even) of 4 pencil pairs, so every bin k = k1 + N1·k2 finds its Hermitian mirror
// N − k in shared memory: k1 = 0 → (0, (N2 − k2) mod N2); k1 = N1/2 → (N1/2, N2 − 1 − k2);
// otherwise (N1 − k1, N2 − 1 − k2).  The forward DIF leaves bin k2 at its digit-reversed position,
// the divide works position by position (reads of both mirrors, CTA barrier, writes), and the
// inverse DIT takes exactly that order back to natural n2: Y is read and written once, in place,
// instead of three round trips through X.
// MP pencil pairs per group (4: 160 KB, one CTA per SM; 2: 80 KB, two per SM)
template <int MP>
__host__ __device__ constexpr size_t mx_fused_tile() { return (size_t)2 * 1024 * (MP + 1) * sizeof(double2); }
template <int MP>
__host__ __device__ constexpr size_t mx_fused_smem() { return mx_fused_tile<MP>() + 2 * 1024 * sizeof(int); }   // + rev2, irev2

template <bool PLAIN, int MP>      // PLAIN: θ = 1 and no λ₃ term, divisor d_k + μ
__global__ void __launch_bounds__(2 * MP * kMxWpp * 32, MP <= 2 ? 2 : 1) k_mx_b_fused(double2* __restrict__ Y, TlongParams Q) {
  constexpr int kMfPairs = MP, kMfRowC = MP + 1, NT = 2 * MP * kMxWpp * 32;
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp / (kMfPairs * kMxWpp), pen = (warp / kMxWpp) % kMfPairs;
  const int t0 = (warp % kMxWpp) * 32 + lane, gid = grp * kMfPairs + pen;
  const int64_t nch4 = (Q.P + kMfPairs - 1) / kMfPairs;
  const int64_t chunk = blockIdx.x % nch4;
  const int j = (int)(blockIdx.x / nch4);
  const int L = Q.N2;
  const bool two = j != 0 || (Q.N1 & 1) == 0;          // does the second group exist
  const int k1b = j == 0 ? Q.N1 / 2 : Q.N1 - j;
  const int ng = two ? 2 : 1;
  for (int idx = threadIdx.x; idx < ng * L * kMfPairs; idx += NT) {
    const int w = idx & (kMfPairs - 1), row = idx / kMfPairs;
    const int g = row >= L ? 1 : 0, n2 = row - g * L;
    const int64_t p = chunk * kMfPairs + w;
    double2* d = sm + (g * L + n2) * kMfRowC + w;
    if (p < Q.P) cp_async16(d, Y + ((int64_t)(g ? k1b : j) * Q.N2 + n2) * Q.P + p);
    else *d = make_double2(0.0, 0.0);
  }
  cp_async_commit();
  int* rs = reinterpret_cast<int*>(reinterpret_cast<char*>(sm) + mx_fused_tile<MP>());
  int* irs = rs + 1024;
#pragma unroll 4
  for (int q = threadIdx.x; q < L; q += NT) {
    rs[q] = __ldg(Q.rev2 + q);
    irs[q] = __ldg(Q.irev2 + q);
  }
  cp_async_wait_all();
  __syncthreads();
  const bool real_pen = chunk * kMfPairs + pen < Q.P && (grp == 0 || two);
  if (real_pen) mix_fft_fwd(sm + grp * L * kMfRowC + pen, kMfRowC, L, Q.plan2, Q.nst2, Q.mt2, t0, gid);
  __syncthreads();
  // Step (2) at every staged position: reads of the element and its mirror into registers first
  constexpr int kPer = (2 * 1024 * kMfPairs + NT - 1) / NT;   // 16
  double2 nv[kPer];
  const double jbar = Q.T.kind >= 2 ? Q.T.st->jbar : 0.0;
  // the pair column w = idx mod MP is the same for all of a thread's elements (NT is a multiple
  // of MP): its two modes' eigenvalues once per thread
  const int64_t p_t = chunk * kMfPairs + (threadIdx.x & (kMfPairs - 1));
  const int64_t sa_t = 2 * p_t, sb_t = sa_t + 1;
  const bool hb_t = sb_t < Q.ns, real_t = p_t < Q.P;
  const double mua = real_t ? mode_mu(sa_t, Q.T, jbar) : 0.0;
  const double mub = real_t && hb_t ? mode_mu(sb_t, Q.T, jbar) : mua;
  const double lama = real_t && Q.T.l3 ? mode_lam(sa_t, Q.T) : 0.0;
  const double lamb = real_t && Q.T.l3 && hb_t ? mode_lam(sb_t, Q.T) : 0.0;
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int idx = threadIdx.x + r * NT;
    nv[r] = make_double2(0.0, 0.0);
    if (idx >= ng * L * kMfPairs) continue;
    const int w = idx & (kMfPairs - 1), row = idx / kMfPairs;
    const int g = row >= L ? 1 : 0, pos = row - g * L;
    const int64_t p = chunk * kMfPairs + w;
    if (p >= Q.P) continue;
    const int k1 = g ? k1b : j;
    const int k2 = rs[pos];
    int mg, k2m;
    if (k1 == 0) { mg = g; k2m = k2 == 0 ? 0 : L - k2; }
    else if (2 * k1 == Q.N1) { mg = g; k2m = L - 1 - k2; }
    else { mg = 1 - g; k2m = L - 1 - k2; }
    const double2 Zl = sm[(g * L + pos) * kMfRowC + w];
    const double2 Zm = sm[(mg * L + irs[k2m]) * kMfRowC + w];
    const double2 A = make_double2(0.5 * (Zl.x + Zm.x), 0.5 * (Zl.y - Zm.y));
    const double2 B = make_double2(0.5 * (Zl.y + Zm.y), -0.5 * (Zl.x - Zm.x));
    const int k = k1 + Q.N1 * k2;
    const double2 d = __ldg(Q.T.dl + k);
    double2 Af, Bf;
    if (PLAIN) {
      Af = cmul(A, cinv_fast(make_double2(d.x + mua, d.y)));
      Bf = cmul(B, cinv_fast(make_double2(d.x + mub, d.y)));
    } else {
      Af = cmul(A, cinv_fast(shifted(d, Q.T.el, k, mua, Q.T.l3, lama)));
      Bf = cmul(B, cinv_fast(shifted(d, Q.T.el, k, mub, Q.T.l3, lamb)));
    }
    nv[r] = make_double2(Af.x - Bf.y, Af.y + Bf.x);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int idx = threadIdx.x + r * NT;
    if (idx >= ng * L * kMfPairs) continue;
    const int w = idx & (kMfPairs - 1), row = idx / kMfPairs;
    const int g = row >= L ? 1 : 0, pos = row - g * L;
    sm[(g * L + pos) * kMfRowC + w] = nv[r];
  }
  __syncthreads();
  if (real_pen) mix_fft_inv(sm + grp * L * kMfRowC + pen, kMfRowC, L, Q.plan2, Q.nst2, Q.mt2, t0, gid);
  __syncthreads();
  for (int idx = threadIdx.x; idx < ng * L * kMfPairs; idx += NT) {
    const int w = idx & (kMfPairs - 1), row = idx / kMfPairs;
    const int g = row >= L ? 1 : 0, n2 = row - g * L;
    const int64_t p = chunk * kMfPairs + w;
    if (p < Q.P) Y[((int64_t)(g ? k1b : j) * Q.N2 + n2) * Q.P + p] = sm[(g * L + n2) * kMfRowC + w];
  }
}

}  // namespace pd
