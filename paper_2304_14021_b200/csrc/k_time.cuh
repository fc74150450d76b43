// k_time.cuh — Steps (1) and (3) along time, and in 2D the fused Step-(2) divide.
//
// Two real time pencils (spatial points s, s+1) are packed into one complex pencil
// z_j = γ_j (r_j[s] + i r_j[s+1]) (γ_j = α^{j/N_t}, R#2); after the forward DFT (DIF, bit-reversed)
// the two Hermitian spectra separate as A_l = (Z_l + conj Z_{N-l})/2, B_l = (Z_l - conj Z_{N-l})/2i.
// 2D: both are divided by their mode's shifted eigenvalue (d_l + μ_pq, or the CH determinant
// d_l - J̄Λ + ε²Λ², R#8), recombined X_l = A_l/den_a + i B_l/den_b and inverse transformed
// (DIT, natural order); the outputs are scaled by γ_j⁻¹ times all normalisations (1/N_t and the
// spatial 1/(2m)²).  Because the spatial DCT/DST passes commute with the time transforms
// (both act on different tensor factors), the time pass runs on spatially transformed data, so each
// pencil is one spatial mode (p, q) and Step-(2) becomes a per-mode divide.
// 1D: the forward half writes the half spectrum [N_x][N_t/2+1] for the pentadiagonal solves and
// the inverse half reads it back.
#pragma once
#include "common.cuh"
#include "fft.cuh"

namespace pd {

struct TimeParams {
  int nt, log2nt;
  int64_t ns;            // spatial points = pencils
  int nx;                // mode index p = s % nx, q = s / nx
  const double* gam;     // γ_j
  const double* ginv;    // scale / γ_j
  const double2* dl;     // d_l = (1 - z ω^l)/Δt, l = 0..nt-1
  const double2* el;     // e_l = θ + (1-θ) z ω^l (θ-method); NULL for θ = 1 (e_l = 1)
  const double2* l3;     // λ_{3,l} = z ω^l (PinT-II): divisor gains λ_{3,l}·Λ; NULL otherwise
  const double* lamx;    // Laplacian eigenvalues along x (and y: same table, square grids)
  int kind;              // 0 biharmonic, 1 linear CH, 2 CH
  double b2, e2;
  const DevStats* st;    // J̄ for CH
  const double2* tw;
  int twlog;
  unsigned long long* amax;   // optional max |out|
  int tune;                   // PARADIAG_TUNE bits (A/B switches for measurements; 0 = defaults)
  int xoff;                   // column slab (multi-rank): global x of local column 0
  int gamma_folded;           // k_time2d_v2: Γ_α and Γ_α⁻¹·(normalisation) applied by the y passes
  int stagger_ns;             // k_time2d_v2: start delay of the second CTA of each SM (phase offset)
};

// shifted eigenvalue d_l + e_l μ of the Step-(2) system; PinT-II adds λ_{3,l}Λ
// — pass lam = Λ of the mode with l3 != NULL
PD_DEV double2 shifted(double2 d, const double2* el, int l, double mu, const double2* l3 = nullptr,
                       double lam = 0.0) {
  double2 s;
  if (!el) {
    s = make_double2(d.x + mu, d.y);
  } else {
    const double2 e = __ldg(el + l);
    s = make_double2(d.x + e.x * mu, d.y + e.y * mu);
  }
  if (l3) {
    const double2 w = __ldg(l3 + l);
    s = make_double2(s.x + w.x * lam, s.y + w.y * lam);
  }
  return s;
}

// Laplacian eigenvalue Λ = λ_p + λ_q of spatial mode s
PD_DEV double mode_lam(int64_t s, const TimeParams& P) {
  const int64_t q = s / P.nx, p = s - q * P.nx;
  return __ldg(P.lamx + P.xoff + p) + (P.nx == P.ns ? 0.0 : __ldg(P.lamx + q));
}

PD_DEV double mode_mu(int64_t s, const TimeParams& P, double jbar) {
  const int64_t q = s / P.nx, p = s - q * P.nx;
  const double Lam = __ldg(P.lamx + P.xoff + p) + (P.nx == P.ns ? 0.0 : __ldg(P.lamx + q));
  if (P.kind == 0) return Lam * Lam;
  if (P.kind == 1) return P.b2 * Lam + P.e2 * (Lam * Lam);
  return -jbar * Lam + P.e2 * (Lam * Lam);          // CH PinT-I (J̄ = mean(3U²-1)) / PinT-II (J̄₃)
}

// Stage the tile's pencil pairs in shared memory with cp.async (natural time order; the
// γ_j scaling is applied on the fly by the first FFT pass).  Points past ns are zero.
template <int NWARP>
PD_DEV void load_pairs(const double* __restrict__ in, double2* smem, int64_t s0, const TimeParams& P) {
  const int pitch = padded16(P.nt);
  double* sd = reinterpret_cast<double*>(smem);
  for (int idx = threadIdx.x; idx < 2 * NWARP * P.nt; idx += NWARP * 32) {
    const int j = idx / (2 * NWARP), rem = idx - j * (2 * NWARP);
    const int w = rem >> 1, c = rem & 1;
    const int64_t s = s0 + rem;
    double* d = sd + 2 * (w * pitch + pad16(j)) + c;
    if (s < P.ns) cp_async8(d, in + (size_t)j * P.ns + s);
    else *d = 0.0;
  }
  cp_async_commit();
  cp_async_wait_all();
}

// Write the tile back (outputs already scaled by the last FFT pass).
template <int NWARP>
PD_DEV void store_pairs(double* __restrict__ out, const double2* smem, int64_t s0, const TimeParams& P) {
  const int pitch = padded16(P.nt);
  const double* sd = reinterpret_cast<const double*>(smem);
  double lmax = 0.0;
  for (int idx = threadIdx.x; idx < 2 * NWARP * P.nt; idx += NWARP * 32) {
    const int j = idx / (2 * NWARP), rem = idx - j * (2 * NWARP);
    const int w = rem >> 1, c = rem & 1;
    const int64_t s = s0 + rem;
    if (s < P.ns) {
      const double v = sd[2 * (w * pitch + pad16(j)) + c];
      out[(size_t)j * P.ns + s] = v;
      lmax = fmax(lmax, fabs(v));
    }
  }
  if (P.amax) warp_atomic_max_abs(P.amax, lmax);
}

// 2D fused time pass: γ-scale, DFT, per-mode divide, inverse DFT, γ⁻¹-scale.  One warp per pair.
template <int NWARP>
__global__ void __launch_bounds__(NWARP * 32)
k_time_solve_2d(const double* in, double* out, TimeParams P) {
  extern __shared__ double2 smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s0 = (int64_t)blockIdx.x * (2 * NWARP);
  load_pairs<NWARP>(in, smem, s0, P);
  __syncthreads();
  double2* buf = smem + warp * padded16(P.nt);
  const int64_t sa = s0 + 2 * warp;
  if (sa < P.ns) {
    warp_fft_dif<-1>(buf, P.log2nt, P.tw, P.twlog, lane, P.gam);
    const double jbar = P.kind >= 2 ? P.st->jbar : 0.0;
    const double mua = mode_mu(sa, P, jbar);
    const double mub = sa + 1 < P.ns ? mode_mu(sa + 1, P, jbar) : mua;
    const int N = P.nt, half = N >> 1;
    for (int l = lane; l <= half; l += 32) {
      const int pl = pad16(bitrev(l, P.log2nt));
      const int m = (N - l) & (N - 1);
      const int pm = pad16(bitrev(m, P.log2nt));
      const double2 Zl = buf[pl], Zm = buf[pm];
      const double2 A = make_double2(0.5 * (Zl.x + Zm.x), 0.5 * (Zl.y - Zm.y));
      const double2 B = make_double2(0.5 * (Zl.y + Zm.y), -0.5 * (Zl.x - Zm.x));
      const double2 d = __ldg(P.dl + l);
      const double2 fa = cinv(shifted(d, P.el, l, mua, P.l3, P.l3 ? mode_lam(sa, P) : 0.0));
      const double2 fb = cinv(shifted(d, P.el, l, mub, P.l3, P.l3 && sa + 1 < P.ns ? mode_lam(sa + 1, P) : 0.0));
      const double2 Af = cmul(A, fa), Bf = cmul(B, fb);
      // X_l = Af + i Bf ; X_{N-l} = conj(Af) + i conj(Bf)
      buf[pl] = make_double2(Af.x - Bf.y, Af.y + Bf.x);
      if (m != l) buf[pm] = make_double2(Af.x + Bf.y, Bf.x - Af.y);
    }
    __syncwarp();
    warp_fft_dit<+1>(buf, P.log2nt, P.tw, P.twlog, lane, P.ginv);
  }
  __syncthreads();
  store_pairs<NWARP>(out, smem, s0, P);
}

// 1D forward: γ-scale + DFT, write the half spectra spec[s][l], l = 0..nt/2.
template <int NWARP>
__global__ void __launch_bounds__(NWARP * 32)
k_time_fwd_1d(const double* in, double2* spec, TimeParams P) {
  extern __shared__ double2 smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s0 = (int64_t)blockIdx.x * (2 * NWARP);
  load_pairs<NWARP>(in, smem, s0, P);
  __syncthreads();
  double2* buf = smem + warp * padded16(P.nt);
  const int64_t sa = s0 + 2 * warp;
  if (sa >= P.ns) return;
  warp_fft_dif<-1>(buf, P.log2nt, P.tw, P.twlog, lane, P.gam);
  const int N = P.nt, half = N >> 1, nb = half + 1;
  for (int l = lane; l <= half; l += 32) {
    const double2 Zl = buf[pad16(bitrev(l, P.log2nt))];
    const double2 Zm = buf[pad16(bitrev((N - l) & (N - 1), P.log2nt))];
    spec[sa * nb + l] = make_double2(0.5 * (Zl.x + Zm.x), 0.5 * (Zl.y - Zm.y));
    if (sa + 1 < P.ns) spec[(sa + 1) * nb + l] = make_double2(0.5 * (Zl.y + Zm.y), -0.5 * (Zl.x - Zm.x));
  }
}

// 1D inverse: read the half spectra of a pencil pair, inverse DFT, γ⁻¹-scale, store.
template <int NWARP>
__global__ void __launch_bounds__(NWARP * 32)
k_time_inv_1d(const double2* spec, double* out, TimeParams P) {
  extern __shared__ double2 smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s0 = (int64_t)blockIdx.x * (2 * NWARP);
  double2* buf = smem + warp * padded16(P.nt);
  const int64_t sa = s0 + 2 * warp;
  if (sa < P.ns) {
    const int N = P.nt, half = N >> 1, nb = half + 1;
    for (int l = lane; l <= half; l += 32) {
      const double2 A = spec[sa * nb + l];
      const double2 B = sa + 1 < P.ns ? spec[(sa + 1) * nb + l] : make_double2(0.0, 0.0);
      const int m = (N - l) & (N - 1);
      buf[pad16(bitrev(l, P.log2nt))] = make_double2(A.x - B.y, A.y + B.x);
      if (m != l) buf[pad16(bitrev(m, P.log2nt))] = make_double2(A.x + B.y, B.x - A.y);
    }
    __syncwarp();
    warp_fft_dit<+1>(buf, P.log2nt, P.tw, P.twlog, lane, P.ginv);
  }
  __syncthreads();
  store_pairs<NWARP>(out, smem, s0, P);
}

}  // namespace pd
