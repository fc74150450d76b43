// fft4.cuh — register-resident warp FFT, "four-step" form, for transform sizes N = 32·E
// (E = 1..32).  One warp holds 1024 complex values: P = 32/E independent transforms.
//
// Layouts (lane = 0..31, 32 registers v[0..31] of double2 per lane):
//   stage-1 layout:  lane l holds x_p[l + 32 e] in v[p·E + e]          (p < P, e < E)
//   stage-2 layout:  lane L = p·E + k1 holds X_p[k1 + E k2] in v[k2]   (k2 < 32)
// Forward:  X[k1 + E k2] = Σ_l W_32^{l k2} [ W_N^{l k1} Σ_e W_E^{e k1} x[l + 32e] ]
//   = E-point DFTs in registers, twiddle, one shared-memory transpose, 32-point DFTs in registers.
// Inverse (stage-2 in, stage-1 out) runs the same steps backwards with conjugate roots, so a
// forward/inverse pair needs exactly two shared-memory round trips and no bit reversal.
// Sign convention (R#1): SIGN = -1 forward exp(-2πi jk/N), +1 inverse (unnormalised).
#pragma once
#include "common.cuh"

namespace pd {

// cos(2πk/32)
__host__ __device__ constexpr double cos32(int k) {
  constexpr double c[8] = {1.0, 0.98078528040323044913, 0.92387953251128675613, 0.83146961230254523708,
                           0.70710678118654752440, 0.55557023301960222474, 0.38268343236508977173,
                           0.19509032201612826785};
  k &= 31;
  // cos is even and cos(π - x) = -cos(x); reduce to the first octant of the table
  const int q = k >> 3, r = k & 7;
  return q == 0 ? c[r] : q == 1 ? (r == 0 ? 0.0 : -c[8 - r]) : q == 2 ? -c[r] : (r == 0 ? 0.0 : c[8 - r]);
}
__host__ __device__ constexpr double sin32(int k) { return cos32(k - 8); }

// v · exp(SIGN·2πi K/32), K compile-time; trivial and (±1±i)/√2 roots specialised.
template <int K, int SIGN>
PD_DEV double2 mul_w32(double2 v) {
  constexpr int k = K & 31;
  if constexpr (k == 0) {
    return v;
  } else if constexpr (k == 8) {
    return SIGN < 0 ? make_double2(v.y, -v.x) : make_double2(-v.y, v.x);
  } else if constexpr (k == 16) {
    return make_double2(-v.x, -v.y);
  } else if constexpr (k == 24) {
    return SIGN < 0 ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
  } else if constexpr ((k & 7) == 4) {
    constexpr double c = cos32(k), s = SIGN * sin32(k);
    constexpr double r = 0.70710678118654752440;
    if constexpr (c > 0 && s > 0) return make_double2((v.x - v.y) * r, (v.x + v.y) * r);
    else if constexpr (c > 0 && s < 0) return make_double2((v.x + v.y) * r, (v.y - v.x) * r);
    else if constexpr (c < 0 && s > 0) return make_double2(-(v.x + v.y) * r, (v.x - v.y) * r);
    else return make_double2((v.y - v.x) * r, -(v.x + v.y) * r);
  } else {
    constexpr double c = cos32(k), s = SIGN * sin32(k);
    return make_double2(v.x * c - v.y * s, v.x * s + v.y * c);
  }
}

template <int SIGN, int K = 0>
PD_DEV double2 mul_w32_rt(double2 v, int k) {
  if constexpr (K == 32) {
    return v;
  } else {
    if (k == K) return mul_w32<K, SIGN>(v);
    return mul_w32_rt<SIGN, K + 1>(v, k);
  }
}

__host__ __device__ constexpr int brev_c(int t, int r) {
  int o = 0;
  for (int i = 0; i < r; ++i) o |= ((t >> i) & 1) << (r - 1 - i);
  return o;
}
__host__ __device__ constexpr int ilog2_c(int v) { return v <= 1 ? 0 : 1 + ilog2_c(v >> 1); }

// R-point DFT in registers (R ≤ 32), natural order in and out.
template <int R, int SIGN>
PD_DEV void dft_reg(double2* v) {
  if constexpr (R == 1) {
    return;
  } else {
#pragma unroll
    for (int half = R / 2; half >= 1; half >>= 1) {
#pragma unroll
      for (int t = 0; t < R; ++t) {
        if (t & half) continue;
        const int m = t & (half - 1);
        const double2 a = v[t], c = v[t + half];
        v[t] = cadd(a, c);
        v[t + half] = mul_w32_rt<SIGN>(csub(a, c), m * (16 / half));
      }
    }
    // DIF leaves the output bit-reversed: undo with compile-time swaps (register renaming)
    constexpr int r = ilog2_c(R);
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const int u = brev_c(t, r);
      if (u > t) {
        const double2 tmp = v[t];
        v[t] = v[u];
        v[u] = tmp;
      }
    }
  }
}

// Powers w^k, k < K (K ≤ 32), of w = W_N^{base} (conjugated for SIGN = +1), from the table
// tw[j] = exp(-2πi j/2^twlog): w^{1,2,4} and w^{8,16} are loaded exactly, w^k = lo[k&7]·hi[k>>3]
// with lo/hi composed by at most one multiply — every power carries ≤ 3 roundings.
template <int K, int SIGN, bool SMEMTAB = false>
struct TwPow {
  static constexpr int NL = K < 8 ? K : 8;
  static constexpr int NH = K <= 8 ? 1 : K / 8;
  double2 lo[NL];
  double2 hi[NH];
  PD_DEV double2 ld(const double2* __restrict__ tw, int e, int N, int sh) {
    double2 t = SMEMTAB ? tw[(e & (N - 1)) << sh] : __ldg(tw + ((e & (N - 1)) << sh));
    if (SIGN > 0) t.y = -t.y;
    return t;
  }
  PD_DEV TwPow(int base, int log2N, const double2* __restrict__ tw, int twlog) {
    const int N = 1 << log2N, sh = twlog - log2N;
    lo[0] = make_double2(1.0, 0.0);
#pragma unroll
    for (int k = 1; k < NL; ++k) {
      if ((k & (k - 1)) == 0) lo[k] = ld(tw, base * k, N, sh);
      else lo[k] = cmul(lo[k - (k & -k)], lo[k & -k]);
    }
    hi[0] = make_double2(1.0, 0.0);
#pragma unroll
    for (int h = 1; h < NH; ++h) {
      if ((h & (h - 1)) == 0) hi[h] = ld(tw, base * 8 * h, N, sh);
      else hi[h] = cmul(hi[h - (h & -h)], hi[h & -h]);
    }
  }
  // v · w^k (k compile-time after unrolling)
  PD_DEV double2 apply(double2 v, int k) const {
    if (k == 0) return v;
    const double2 a = cmul(v, lo[k & 7 & (NL - 1)]);
    return (k >> 3) ? cmul(a, hi[(k >> 3) & (NH - 1)]) : a;
  }
};

PD_DEV int tpad(int q) { return q + (q >> 5); }
constexpr int kWarpScratch = 1024 + 32;   // complex slots per warp (tpad(1023) = 1054)

// Forward (SIGN=-1) or inverse-direction (SIGN=+1) transform: stage-1 layout in, stage-2 out.
template <int E, int SIGN, bool SMEMTAB = false>
PD_DEV void fft4_s1_to_s2(double2 (&v)[32], double2* T, int log2N, const double2* __restrict__ tw,
                          int twlog, int lane) {
  constexpr int P = 32 / E;
  const TwPow<E, SIGN, SMEMTAB> w(lane, log2N, tw, twlog);           // W_N^{l·k1}, l = lane
#pragma unroll
  for (int p = 0; p < P; ++p) {
    dft_reg<E, SIGN>(v + p * E);
#pragma unroll
    for (int k1 = 0; k1 < E; ++k1) T[tpad((p * E + k1) * 32 + lane)] = w.apply(v[p * E + k1], k1);
  }
  __syncwarp();
#pragma unroll
  for (int l = 0; l < 32; ++l) v[l] = T[tpad(lane * 32 + l)];
  __syncwarp();
  dft_reg<32, SIGN>(v);
}

// Stage-2 layout in, stage-1 layout out (the reverse of fft4_s1_to_s2 with the same SIGN
// convention for its roots).  Used with SIGN=+1 to invert a forward transform.
template <int E, int SIGN, bool SMEMTAB = false>
PD_DEV void fft4_s2_to_s1(double2 (&v)[32], double2* T, int log2N, const double2* __restrict__ tw,
                          int twlog, int lane) {
  constexpr int P = 32 / E;
  dft_reg<32, SIGN>(v);                                     // over k2 -> index l
  {
    const TwPow<32, SIGN, SMEMTAB> w(lane % E, log2N, tw, twlog);    // W_N^{l·k1}, l = register index
#pragma unroll
    for (int l = 0; l < 32; ++l) T[tpad(lane * 32 + l)] = w.apply(v[l], l);
  }
  __syncwarp();
#pragma unroll
  for (int p = 0; p < P; ++p) {
#pragma unroll
    for (int k = 0; k < E; ++k) v[p * E + k] = T[tpad((p * E + k) * 32 + lane)];
    dft_reg<E, SIGN>(v + p * E);
  }
  __syncwarp();
}

}  // namespace pd
