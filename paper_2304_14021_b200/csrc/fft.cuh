// fft.cuh — warp-level in-place complex FFT on shared memory, radix-2^r (r ≤ 4) passes.
//
// Forward transforms are decimation-in-frequency (natural order in, bit-reversed order out);
// the inverse is decimation-in-time (bit-reversed in, natural out), so a forward/inverse pair
// never needs a separate bit-reversal permutation.  Each pass loads R = 2^r elements with
// stride Q = H/R from a group of size H, runs an R-point DFT in registers with compile-time
// twiddles, and applies the inter-pass twiddles W_H^{j·rev_r(t)} from a global table
// tw[k] = exp(-2πi k / 2^twlog) (L1-resident).  Passes of one transform touch disjoint
// elements per lane, so only __syncwarp() separates them.
//
// Sign convention (R#1): forward = exp(-2πi jk/N); SIGN = -1 forward, +1 inverse (unnormalised).
#pragma once
#include "common.cuh"

namespace pd {

// cos / sin of 2πk/16
__host__ __device__ constexpr double cos16(int k) {
  return k == 0 ? 1.0 : k == 1 ? 0.92387953251128675613 : k == 2 ? 0.70710678118654752440
       : k == 3 ? 0.38268343236508977173 : k == 4 ? 0.0 : k == 5 ? -0.38268343236508977173
       : k == 6 ? -0.70710678118654752440 : k == 7 ? -0.92387953251128675613 : k == 8 ? -1.0
       : k == 9 ? -0.92387953251128675613 : k == 10 ? -0.70710678118654752440
       : k == 11 ? -0.38268343236508977173 : k == 12 ? 0.0 : k == 13 ? 0.38268343236508977173
       : k == 14 ? 0.70710678118654752440 : 0.92387953251128675613;
}
__host__ __device__ constexpr double sin16(int k) { return cos16((k + 12) & 15); }

// v * exp(SIGN * 2πi K / 16), K compile-time
template <int K, int SIGN>
PD_DEV double2 mul_w16(double2 v) {
  if constexpr (K == 0) {
    return v;
  } else if constexpr (K == 4) {
    return SIGN < 0 ? make_double2(v.y, -v.x) : make_double2(-v.y, v.x);
  } else if constexpr (K == 8) {
    return make_double2(-v.x, -v.y);
  } else if constexpr (K == 12) {
    return SIGN < 0 ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
  } else if constexpr (K == 2 || K == 6 || K == 10 || K == 14) {
    // (±1 ± i)/√2 : two adds and two muls
    constexpr double c = cos16(K), s = SIGN * sin16(K);
    constexpr double r = 0.70710678118654752440;
    if constexpr (c > 0 && s > 0) return make_double2((v.x - v.y) * r, (v.x + v.y) * r);
    else if constexpr (c > 0 && s < 0) return make_double2((v.x + v.y) * r, (v.y - v.x) * r);
    else if constexpr (c < 0 && s > 0) return make_double2(-(v.x + v.y) * r, (v.x - v.y) * r);
    else return make_double2((v.y - v.x) * r, -(v.x + v.y) * r);
  } else {
    constexpr double c = cos16(K), s = SIGN * sin16(K);
    return make_double2(v.x * c - v.y * s, v.x * s + v.y * c);
  }
}

template <int SIGN>
PD_DEV double2 mul_w16_rt(double2 v, int k) {
  switch (k & 15) {
    case 0: return mul_w16<0, SIGN>(v);   case 1: return mul_w16<1, SIGN>(v);
    case 2: return mul_w16<2, SIGN>(v);   case 3: return mul_w16<3, SIGN>(v);
    case 4: return mul_w16<4, SIGN>(v);   case 5: return mul_w16<5, SIGN>(v);
    case 6: return mul_w16<6, SIGN>(v);   case 7: return mul_w16<7, SIGN>(v);
    case 8: return mul_w16<8, SIGN>(v);   case 9: return mul_w16<9, SIGN>(v);
    case 10: return mul_w16<10, SIGN>(v); case 11: return mul_w16<11, SIGN>(v);
    case 12: return mul_w16<12, SIGN>(v); case 13: return mul_w16<13, SIGN>(v);
    case 14: return mul_w16<14, SIGN>(v); default: return mul_w16<15, SIGN>(v);
  }
}

__host__ __device__ constexpr int rev_const(int t, int r) {
  int o = 0;
  for (int i = 0; i < r; ++i) o |= ((t >> i) & 1) << (r - 1 - i);
  return o;
}

// R-point DFT in registers, natural in -> bit-reversed out (radix-2 DIF stages).
template <int R, int SIGN>
PD_DEV void dif_reg(double2 (&v)[R]) {
#pragma unroll
  for (int half = R / 2; half >= 1; half >>= 1) {
#pragma unroll
    for (int t = 0; t < R; ++t) {
      if (t & half) continue;
      const int m = t & (half - 1);
      const double2 a = v[t], c = v[t + half];
      v[t] = cadd(a, c);
      v[t + half] = mul_w16_rt<SIGN>(csub(a, c), m * (8 / half));
    }
  }
}

// R-point DFT in registers, bit-reversed in -> natural out (radix-2 DIT stages).
template <int R, int SIGN>
PD_DEV void dit_reg(double2 (&v)[R]) {
#pragma unroll
  for (int half = 1; half < R; half <<= 1) {
#pragma unroll
    for (int t = 0; t < R; ++t) {
      if (t & half) continue;
      const int m = t & (half - 1);
      const double2 a = v[t], c = mul_w16_rt<SIGN>(v[t + half], m * (8 / half));
      v[t] = cadd(a, c);
      v[t + half] = csub(a, c);
    }
  }
}

template <int SIGN>
PD_DEV double2 twiddle(const double2* __restrict__ tw, int idx) {
  double2 w = __ldg(tw + idx);
  if (SIGN > 0) w.y = -w.y;
  return w;
}

// One DIF pass of radix R = 2^r on a transform of size N = 2^log2n starting at stage s.
template <int r, int SIGN>
PD_DEV void dif_pass(double2* buf, int log2n, int s, const double2* __restrict__ tw, int twlog,
                     int lane, const double* __restrict__ pre = nullptr) {
  constexpr int R = 1 << r;
  const int log2H = log2n - s, log2Q = log2H - r;
  const int H = 1 << log2H, Q = 1 << log2Q;
  const int nblk = 1 << (log2n - r);
  const int tshift = twlog - log2H;
  for (int b = lane; b < nblk; b += 32) {
    const int g = b >> log2Q, j = b & (Q - 1);
    const int base = (g << log2H) + j;
    double2 v[R];
#pragma unroll
    for (int t = 0; t < R; ++t) v[t] = buf[pad16(base + t * Q)];
    if (pre) {
#pragma unroll
      for (int t = 0; t < R; ++t) v[t] = cscale(v[t], __ldg(pre + base + t * Q));
    }
    dif_reg<R, SIGN>(v);
#pragma unroll
    for (int t = 1; t < R; ++t) {
      const int e = (j * rev_const(t, r)) & (H - 1);
      if (j) v[t] = cmul(v[t], twiddle<SIGN>(tw, e << tshift));
    }
#pragma unroll
    for (int t = 0; t < R; ++t) buf[pad16(base + t * Q)] = v[t];
  }
}

// One DIT pass of radix R = 2^r: sub-transforms of size Q = 2^log2Q are combined into H = R·Q.
template <int r, int SIGN>
PD_DEV void dit_pass(double2* buf, int log2n, int log2Q, const double2* __restrict__ tw, int twlog,
                     int lane, const double* __restrict__ post = nullptr) {
  constexpr int R = 1 << r;
  const int log2H = log2Q + r;
  const int H = 1 << log2H, Q = 1 << log2Q;
  const int nblk = 1 << (log2n - r);
  const int tshift = twlog - log2H;
  for (int b = lane; b < nblk; b += 32) {
    const int g = b >> log2Q, j = b & (Q - 1);
    const int base = (g << log2H) + j;
    double2 v[R];
#pragma unroll
    for (int t = 0; t < R; ++t) v[t] = buf[pad16(base + t * Q)];
#pragma unroll
    for (int t = 1; t < R; ++t) {
      const int e = (j * rev_const(t, r)) & (H - 1);
      if (j) v[t] = cmul(v[t], twiddle<SIGN>(tw, e << tshift));
    }
    dit_reg<R, SIGN>(v);
    if (post) {
#pragma unroll
      for (int t = 0; t < R; ++t) v[t] = cscale(v[t], __ldg(post + base + t * Q));
    }
#pragma unroll
    for (int t = 0; t < R; ++t) buf[pad16(base + t * Q)] = v[t];
  }
}

// Forward (SIGN=-1) or inverse (SIGN=+1) DIF FFT: natural in, bit-reversed out.  `pre`
// (optional, real, natural order) scales the input on the fly in the first pass.
template <int SIGN>
PD_DEV void warp_fft_dif(double2* buf, int log2n, const double2* __restrict__ tw, int twlog, int lane,
                         const double* __restrict__ pre = nullptr) {
  int s = 0;
  while (s < log2n) {
    const int r = min(4, log2n - s);
    const double* p = s == 0 ? pre : nullptr;
    switch (r) {
      case 4: dif_pass<4, SIGN>(buf, log2n, s, tw, twlog, lane, p); break;
      case 3: dif_pass<3, SIGN>(buf, log2n, s, tw, twlog, lane, p); break;
      case 2: dif_pass<2, SIGN>(buf, log2n, s, tw, twlog, lane, p); break;
      default: dif_pass<1, SIGN>(buf, log2n, s, tw, twlog, lane, p); break;
    }
    __syncwarp();
    s += r;
  }
}

// DIT FFT: bit-reversed in, natural out.  The first pass takes the remainder radix so that the
// pass list is the DIF list reversed.
// `post` (optional, real, natural order) scales the output in the last pass.
template <int SIGN>
PD_DEV void warp_fft_dit(double2* buf, int log2n, const double2* __restrict__ tw, int twlog, int lane,
                         const double* __restrict__ post = nullptr) {
  int log2Q = 0;
  int rem = log2n & 3;
  while (log2Q < log2n) {
    const int r = rem ? rem : 4;
    rem = 0;
    const double* p = log2Q + r >= log2n ? post : nullptr;
    switch (r) {
      case 4: dit_pass<4, SIGN>(buf, log2n, log2Q, tw, twlog, lane, p); break;
      case 3: dit_pass<3, SIGN>(buf, log2n, log2Q, tw, twlog, lane, p); break;
      case 2: dit_pass<2, SIGN>(buf, log2n, log2Q, tw, twlog, lane, p); break;
      default: dit_pass<1, SIGN>(buf, log2n, log2Q, tw, twlog, lane, p); break;
    }
    __syncwarp();
    log2Q += r;
  }
}

}  // namespace pd
