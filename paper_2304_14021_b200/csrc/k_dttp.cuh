// k_dttp.cuh — DCT-I / DST-I line transform of length M = 2048 (c5's 2049-node lines) by a PAIR of
// warps (64 threads, 16 complex values per thread), Step-(2) of P:162 in 2D.
//
// Same mathematics as k_dtt.cuh (the M/2-point complex FFT with the pre-/post-processing of
// SURVEY Appendix B).  Why a pair: with one warp per line every lane holds 32 complex values
// (≈250 registers), so only 8 warps fit on an SM and the line kernels are latency bound (ncu d3b:
// IPC 1.1, halving the warps made them 1.5x slower).  Splitting a line over two warps halves the
// registers per thread and doubles the warps per SM.  The 1024-point FFT becomes three register
// stages with two shared-memory transposes:
//   A:  t = 0..63 holds z[t + 64e], e = 0..15      16-point DFT over e, twiddle W_1024^{t k1}
//   B1: (k1, p) = (t/4, t%4) holds A[p + 4m][k1]    16-point DFT over m, twiddle W_64^{p k2}
//   B2: (k1, g) = (t/4, t%4) holds C[k1][p][4g+i]   4-point DFTs over p
// giving Z[k1 + 16(4g + i) + 256 q].  The spectrum is parked in natural order, the split and the
// prefix sums run blocked (thread t owns k = 16t .. 16t+15; one 64-thread scan per line), the
// outputs are staged for coalesced stores.  The two warps of a pair synchronise with a named
// barrier (bar.sync id, 64).
#pragma once
#include "common.cuh"
#include "fft4.cuh"
#include "k_spatial.cuh"

namespace pd {

// Named barrier of one warp pair.  The id must be an immediate: with a register operand ptxas
// reserves all 16 hardware barriers for the CTA, which caps the CTAs per SM.
template <int ID>
PD_DEV void bar_sync64() { asm volatile("bar.sync %0, 64;" ::"n"(ID) : "memory"); }
PD_DEV void pair_sync(int id) {
  switch (id) {
    case 1: bar_sync64<1>(); break;
    case 2: bar_sync64<2>(); break;
    case 3: bar_sync64<3>(); break;
    case 4: bar_sync64<4>(); break;
    case 5: bar_sync64<5>(); break;
    case 6: bar_sync64<6>(); break;
    case 7: bar_sync64<7>(); break;
    default: bar_sync64<8>(); break;
  }
}

template <int NEUMANN>
struct DttPair {
  static constexpr int M = 2048, H = 1024, LDX = M + 2;
  static constexpr int TP = 68;                         // transpose row pitch (≡ 4 mod 8 slots)
  static PD_DEV int ppos(int k) { return k + (k >> 4); }        // park: 1024 + 64 slots
  static PD_DEV int opos(int q) { return q + (q >> 5); }        // output staging: 2049 + 64
  static constexpr int BUF = 2 * 1100;                  // doubles per pair (17.6 KB)
  static_assert(2 * 16 * TP <= BUF && 2 * (H + H / 16) <= BUF && M + 1 + (M >> 5) + 1 <= BUF, "pair buffer");

  // xb: the pair's buffer holding x_0..x_M (hinged ends zero); on return the outputs at opos(q).
  // t = thread in pair (0..63), h = warp in pair, bid = named barrier id, xs = 2-double scratch
  // (cross-warp sums), trig2p[j*64 + t] = (cos, sin)(2π(16t + j)/M).  g scales every output.
  PD_DEV static void transform(double* xb, const LineParams& L, const double2* __restrict__ trig2p, int t,
                               int bid, double* xs, double g = 1.0) {
    const int lane = t & 31, h = t >> 5;
    double2 v[16];
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int n = t + 64 * e, j0 = 2 * n;
      const double2 a = *reinterpret_cast<const double2*>(xb + j0);
      const double m0 = xb[M - j0], m1 = xb[M - j0 - 1];
      const double2 t0 = __ldg(L.trig + j0), t1 = __ldg(L.trig + j0 + 1);
      v[e] = make_double2(ymap<NEUMANN>(a.x, m0, t0.y), ymap<NEUMANN>(a.y, m1, t1.y));
      if (NEUMANN) acc = fma(a.x - m0, t0.x, fma(a.y - m1, t1.x, acc));
    }
    if (NEUMANN) {
      acc = warp_sum(acc);
      if (lane == 0) xs[h] = acc;
    }
    pair_sync(bid);                                      // xb consumed; xs written
    const double x1 = NEUMANN ? xs[0] + xs[1] : 0.0;
    double2* T = reinterpret_cast<double2*>(xb);
    // ---- stage A
    dft_reg<16, -1>(v);
    {
      const TwPow<16, -1> w(t, 10, L.tw, L.twlog);
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) T[k1 * TP + t] = w.apply(v[k1], k1);
    }
    pair_sync(bid);
    const int k1 = t >> 2, p = t & 3;
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = T[k1 * TP + p + 4 * m];
    pair_sync(bid);
    // ---- stage B1: 16-point DFT over m, twiddle W_64^{p k2}
    dft_reg<16, -1>(v);
    {
      const TwPow<16, -1> w(16 * p, 10, L.tw, L.twlog);
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) T[k1 * TP + p * 17 + (k2 & 3) * 4 + (k2 >> 2)] = w.apply(v[k2], k2);
    }
    pair_sync(bid);
    // ---- stage B2: thread (k1, g) — four 4-point DFTs over p (k2 = 4g + i)
    {
      const int gq = p;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double2 u[4];
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) u[pp] = T[k1 * TP + pp * 17 + i * 4 + gq];
        dft_reg<4, -1>(u);
#pragma unroll
        for (int q = 0; q < 4; ++q) v[i * 4 + q] = u[q];       // Z[k1 + 64 g + 16 i + 256 q]
      }
    }
    pair_sync(bid);
    {
      const int gq = p;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) T[ppos(k1 + 64 * gq + 16 * i + 256 * q)] = v[i * 4 + q];
    }
    pair_sync(bid);
    // ---- blocked split + prefix: thread t owns k = 16t + j
    const double g2 = 2.0 * g;
    double run = 0.0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int k = 16 * t + j;
      const double2 Zk = T[ppos(k)];
      const double2 Zm = T[ppos((H - k) & (H - 1))];
      const double2 Ev = make_double2(0.5 * (Zk.x + Zm.x), 0.5 * (Zk.y - Zm.y));
      const double2 O = make_double2(0.5 * (Zk.y + Zm.y), -0.5 * (Zk.x - Zm.x));
      const double2 tw2 = __ldg(trig2p + j * 64 + t);
      const double Yx = Ev.x + tw2.x * O.x + tw2.y * O.y;
      const double Yy = Ev.y + tw2.x * O.y - tw2.y * O.x;
      double ev, a;
      if (NEUMANN) {
        ev = g2 * Yx;
        a = k == 0 ? 0.0 : Yy;
      } else {
        ev = -g2 * Yy;
        a = k == 0 ? g * Yx : g2 * Yx;
      }
      run += a;
      v[j] = make_double2(ev, run);
    }
    const double2 Z0 = T[ppos(0)];
    // exclusive scan of the 64 block totals (warp scan + the first warp's total)
    double incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double tt = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += tt;
    }
    double excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 0.0;
    if (h == 0 && lane == 31) xs[0] = incl;
    pair_sync(bid);                                      // T fully read; warp 0 total visible
    if (h == 1) excl += xs[0];
    const double gx1 = g * x1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int q = 32 * t + 2 * j;
      if (NEUMANN) {
        xb[opos(q)] = v[j].x;                                   // X_{2k}
        xb[opos(q + 1)] = fma(-g2, excl + v[j].y, gx1);         // X_{2k+1}
      } else {
        xb[opos(q)] = excl + v[j].y;                            // X_{2k+1}: stored index 2k
        if (q > 0) xb[opos(q - 1)] = v[j].x;                    // X_{2k}:   stored index 2k-1
      }
    }
    if (NEUMANN && t == 63) xb[opos(M)] = g2 * (Z0.x - Z0.y);  // X_M
    pair_sync(bid);
  }
};

// ---------------------------------------------------------------- rows: independent warp pairs
template <int NEUMANN, int NPAIR>
__global__ void __launch_bounds__(NPAIR * 64, 4)
k_rows4(const double* in, double* out, LineParams L, const double2* __restrict__ trig2p) {
  using D = DttPair<NEUMANN>;
  extern __shared__ double2 smem2[];
  __shared__ double xsum[NPAIR][2];
  const int pair = threadIdx.x >> 6, t = threadIdx.x & 63, lane = threadIdx.x & 31;
  const int bid = 1 + pair;
  double* xb = reinterpret_cast<double*>(smem2) + (size_t)pair * D::BUF;
  double lmax = 0.0;
  const int64_t gstride = (int64_t)gridDim.x * NPAIR;
  for (int64_t line = (int64_t)blockIdx.x * NPAIR + pair; line < L.nlines; line += gstride) {
    const double* src = in + line * L.nx;
    double* x = xb + (NEUMANN ? 0 : 1);
    for (int e = t; e < L.nel; e += 64) cp_async8(x + e, src + e);
    cp_async_commit();
    if (!NEUMANN && t == 0) {
      xb[0] = 0.0;
      xb[D::M] = 0.0;
    }
    cp_async_wait_all();
    pair_sync(bid);
    D::transform(xb, L, trig2p, t, bid, xsum[pair]);
    double* d = out + line * L.nx;
    if (L.amax) {
      for (int q = t; q < L.nel; q += 64) {
        const double v = xb[D::opos(q)];
        d[q] = v;
        lmax = amax_acc(lmax, v);
      }
    } else {
      for (int q = t; q < L.nel; q += 64) d[q] = xb[D::opos(q)];
    }
    pair_sync(bid);
  }
  if (L.amax) {
    unsigned long long b = (unsigned long long)__double_as_longlong(lmax);
    b = warp_max_u64(b);
    if (lane == 0 && b) atomicMax(L.amax, b);
  }
}

// ---------------------------------------------------------------- columns: CTA = 8 pairs
template <int NEUMANN>
__global__ void __launch_bounds__(512, 1)
k_cols4(const double* in, double* out, LineParams L, const double2* __restrict__ trig2p) {
  using D = DttPair<NEUMANN>;
  constexpr int C = 8, NTH = 512, RSTEP = NTH / C;    // 8 columns, 64 rows per sweep
  extern __shared__ double2 smem2[];
  __shared__ double xsum[C][2];
  double* base = reinterpret_cast<double*>(smem2);
  const int pair = threadIdx.x >> 6, t = threadIdx.x & 63, lane = threadIdx.x & 31;
  double* xb = base + (size_t)pair * D::BUF;
  const int64_t gx = (L.nx + C - 1) / C;
  const int64_t nsl = L.nlines / L.nx;
  const int64_t ngroups = nsl * gx;
  double lmax = 0.0;
  const int c_t = threadIdx.x % C, e_t = threadIdx.x / C;
  for (int64_t G = blockIdx.x; G < ngroups; G += gridDim.x) {
    const int64_t n = G / gx;
    const int x0 = (int)((G - n * gx) * C);
    const int wcols = min(C, (int)(L.nx - x0));
    const double* src = in + n * L.ns + x0;
    double* dst = out + n * L.ns + x0;
    if (c_t < wcols) {
      double* lb = base + (size_t)c_t * D::BUF + (NEUMANN ? 0 : 1);
      const double* s = src + (int64_t)e_t * L.nx + c_t;
      const int64_t rstride = (int64_t)RSTEP * L.nx;
      for (int e = e_t; e < L.nel; e += RSTEP, s += rstride) cp_async8(lb + e, s);
    }
    cp_async_commit();
    if (!NEUMANN && t == 0) {
      xb[0] = 0.0;
      xb[D::M] = 0.0;
    }
    cp_async_wait_all();
    __syncthreads();
    D::transform(xb, L, trig2p, t, 1 + pair, xsum[pair], L.oscale ? __ldg(L.oscale + n) : 1.0);
    __syncthreads();
    if (c_t < wcols) {
      const double* ob = base + (size_t)c_t * D::BUF;
      double* d = dst + (int64_t)e_t * L.nx + c_t;
      const int64_t rstride = (int64_t)RSTEP * L.nx;
      if (L.amax) {
        for (int e = e_t; e < L.nel; e += RSTEP, d += rstride) {
          const double v = ob[D::opos(e)];
          *d = v;
          lmax = amax_acc(lmax, v);
        }
      } else {
        for (int e = e_t; e < L.nel; e += RSTEP, d += rstride) *d = ob[D::opos(e)];
      }
    }
    __syncthreads();
  }
  if (L.amax) {
    unsigned long long b = (unsigned long long)__double_as_longlong(lmax);
    b = warp_max_u64(b);
    if (lane == 0 && b) atomicMax(L.amax, b);
  }
}

}  // namespace pd
