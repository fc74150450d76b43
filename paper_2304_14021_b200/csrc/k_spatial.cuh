// k_spatial.cuh — DCT-I (Neumann) / DST-I (hinged) along one axis of every time slice.
//
// Step-(2) of P:162 in 2D diagonalises Δ_h with the unnormalised real-to-real transforms
// (P:233):
//   DCT-I  X_k = x_0 + (-1)^k x_M + 2 Σ_{j=1}^{M-1} x_j cos(πjk/M),   k = 0..M   (Neumann nodes)
//   DST-I  X_k = 2 Σ_{j=1}^{M-1} x_j sin(πjk/M),                        k = 1..M-1 (hinged interior)
// Both are self-inverse up to 2M, so the same kernel serves the forward and inverse passes (the
// 1/(2M) factors are folded into the time pass).  M = m is a power of two.
//
// Algorithm (one warp per line, derivation in DESIGN.md §5): a real sequence y of length M is
// built from x and its mirror (a_j = x_j ± x_{M-j}, b_j = x_j ∓ x_{M-j}, s_j = sin(πj/M)),
// packed as M/2 complex z_n = y_{2n} + i y_{2n+1}, transformed with the warp FFT (DIF, output in
// bit-reversed order), split into the real FFT Y_k = E_k + W_M^k O_k, and the outputs follow as
//   DCT-I: X_{2k} = 2 Re Y_k, X_{2k+1} = X_1 - 2 Σ_{i=1}^{k} Im Y_i, X_1 = Σ_j b_j cos(πj/M)
//   DST-I: X_{2k} = -2 Im Y_k, X_{2k+1} = Re Y_0 + 2 Σ_{i=1}^{k} Re Y_i
// with the prefix sums done by warp scans over the interleaved k layout.
#pragma once
#include "common.cuh"
#include "fft.cuh"

namespace pd {

struct LineParams {
  int64_t nlines;
  int64_t A, B, C;       // base(L) = (L / A)·B + (L % A)·C
  int64_t es;            // element stride along the line
  int M, log2h;          // M = m (intervals); H = M/2 complex points
  const double2* trig;   // trig[j] = (cos(πj/M), sin(πj/M)), j = 0..M
  const double2* tw;     // FFT twiddles exp(-2πik/2^twlog)
  int twlog;
  unsigned long long* amax;   // optional: max |out| (NULL = off)
};

template <int NEUMANN>
__device__ __forceinline__ double line_ld(const double* __restrict__ p, int j, int M, int64_t es) {
  if (NEUMANN) return __ldg(p + (int64_t)j * es);
  return (j == 0 || j == M) ? 0.0 : __ldg(p + (int64_t)(j - 1) * es);
}

// Warp-per-line transform.  in and out may alias (each warp reads its whole line before writing).
template <int NEUMANN, int NWARP>
__global__ void __launch_bounds__(NWARP * 32)
k_dtt_lines(const double* in, double* out, LineParams P) {
  extern __shared__ double2 smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = 1 << P.log2h;
  double2* buf = smem + (size_t)warp * padded16(H);
  const int64_t L = (int64_t)blockIdx.x * NWARP + warp;
  if (L >= P.nlines) return;
  const int64_t base = (L / P.A) * P.B + (L % P.A) * P.C;
  const double* src = in + base;
  double* dst = out + base;
  const int M = P.M;

  // ---- pre-processing: y_j from x_j and the mirror x_{M-j}; DCT-I also X_1
  double x1 = 0.0;
  for (int n = lane; n < H; n += 32) {
    const int j0 = 2 * n, j1 = 2 * n + 1;
    const double xa0 = line_ld<NEUMANN>(src, j0, M, P.es), xb0 = line_ld<NEUMANN>(src, M - j0, M, P.es);
    const double xa1 = line_ld<NEUMANN>(src, j1, M, P.es), xb1 = line_ld<NEUMANN>(src, M - j1, M, P.es);
    const double s0 = __ldg(&P.trig[j0].y), s1 = __ldg(&P.trig[j1].y);
    double y0, y1;
    if (NEUMANN) {
      const double b0 = xa0 - xb0, b1 = xa1 - xb1;
      y0 = 0.5 * (xa0 + xb0) - s0 * b0;
      y1 = 0.5 * (xa1 + xb1) - s1 * b1;
      x1 += b0 * __ldg(&P.trig[j0].x) + b1 * __ldg(&P.trig[j1].x);
    } else {
      y0 = s0 * (xa0 + xb0) + 0.5 * (xa0 - xb0);
      y1 = s1 * (xa1 + xb1) + 0.5 * (xa1 - xb1);
    }
    buf[pad16(n)] = make_double2(y0, y1);
  }
  if (NEUMANN) x1 = warp_sum(x1);
  __syncwarp();

  warp_fft_dif<-1>(buf, P.log2h, P.tw, P.twlog, lane);

  // ---- post-processing: real-FFT split, outputs and the prefix sums
  double carry = 0.0;
  double lmax = 0.0;
  for (int k0 = 0; k0 < H; k0 += 32) {
    const int k = k0 + lane;
    double ev = 0.0, scanv = 0.0;
    if (k < H) {
      const double2 Zk = buf[pad16(bitrev(k, P.log2h))];
      const double2 Zm = buf[pad16(bitrev((H - k) & (H - 1), P.log2h))];
      const double2 E = make_double2(0.5 * (Zk.x + Zm.x), 0.5 * (Zk.y - Zm.y));
      const double2 O = make_double2(0.5 * (Zk.y + Zm.y), -0.5 * (Zk.x - Zm.x));
      const double2 t2 = __ldg(&P.trig[2 * k]);          // W_M^k = cos - i sin
      const double2 Y = make_double2(E.x + t2.x * O.x + t2.y * O.y, E.y + t2.x * O.y - t2.y * O.x);
      if (NEUMANN) {
        ev = 2.0 * Y.x;                                   // X_{2k}
        scanv = k == 0 ? 0.0 : Y.y;
      } else {
        ev = -2.0 * Y.y;                                  // X_{2k} (k ≥ 1)
        scanv = k == 0 ? Y.x : 2.0 * Y.x;
      }
    }
    // inclusive warp scan of scanv
    double incl = scanv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const double S = carry + incl;
    carry += __shfl_sync(0xffffffffu, incl, 31);
    if (k < H) {
      if (NEUMANN) {
        const double odd = x1 - 2.0 * S;                  // X_{2k+1}
        dst[(int64_t)(2 * k) * P.es] = ev;
        dst[(int64_t)(2 * k + 1) * P.es] = odd;
        lmax = fmax(lmax, fmax(fabs(ev), fabs(odd)));
      } else {
        dst[(int64_t)(2 * k) * P.es] = S;                 // X_{2k+1} at memory index 2k
        if (k > 0) dst[(int64_t)(2 * k - 1) * P.es] = ev; // X_{2k} at memory index 2k-1
        lmax = fmax(lmax, fmax(fabs(ev), fabs(S)));
      }
    }
  }
  if (NEUMANN && lane == 0) {
    const double2 Z0 = buf[pad16(0)];
    const double xm = 2.0 * (Z0.x - Z0.y);                // X_M = 2 Re Y_{M/2}
    dst[(int64_t)M * P.es] = xm;
    lmax = fmax(lmax, fabs(xm));
  }
  if (P.amax) warp_atomic_max_abs(P.amax, lmax);
}

}  // namespace pd
