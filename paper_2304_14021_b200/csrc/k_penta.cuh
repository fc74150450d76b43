// k_penta.cuh — 1D Step-(2): for every frequency bin l, solve the complex pentadiagonal
// system (d_l I + e_l A) x = ŝ_l (e_l = θ + (1-θ) z ω^l, = 1 for θ = 1) by LU without pivoting plus
// one refinement step whose
// residual uses the nested operator A x = L(L x) or β² L x + ε² L(L x) (R#15; SURVEY probe p10).
// One thread per bin; bins are the fastest-varying index of spec[x][l] so loads coalesce.
#pragma once
#include "common.cuh"

namespace pd {

struct PentaParams {
  int n;                 // unknowns
  int nb;                // bins = nt/2 + 1
  int neumann;
  int kind;              // 0 biharmonic, 1 linear CH
  double inv_h2, b2, e2;
  const double* band;    // 5 x n real bands of assembled A: [a2 | a1 | a0 | c1 | c2]
  const double2* dl;     // d_l
  const double2* el;     // e_l (NULL: θ = 1, e_l = 1)
  double2 *l1, *l2, *iu0, *u1;   // factors [n][nb]
  int refine;            // refinement cap (kPentaRefine; PARADIAG_PENTA_REFINE for A/B)
};

// LU factorisation of d_l I + A (no pivoting), one thread per bin.  Done once at init.
__global__ void k_penta_factor(PentaParams P) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= P.nb) return;
  const double2 d = P.dl[l];
  const double2 e = P.el ? P.el[l] : make_double2(1.0, 0.0);
  const int n = P.n;
  const double* a2 = P.band;
  const double* a1 = P.band + n;
  const double* a0 = P.band + 2 * n;
  const double* c1 = P.band + 3 * n;
  const double* c2 = P.band + 4 * n;
  double2 u0m1 = {0, 0}, u0m2 = {0, 0}, u1m1 = {0, 0}, u1m2 = {0, 0};
  double2 u2m1 = {0, 0}, u2m2 = {0, 0};
  for (int i = 0; i < n; ++i) {
    double2 L2 = {0, 0}, L1 = {0, 0};
    if (i >= 2) L2 = cmul(cscale(e, a2[i]), cinv(u0m2));
    if (i >= 1) {
      double2 num = cscale(e, a1[i]);
      if (i >= 2) num = csub(num, cmul(L2, u1m2));
      L1 = cmul(num, cinv(u0m1));
    }
    double2 U0 = cadd(d, cscale(e, a0[i]));
    if (i >= 2) U0 = csub(U0, cmul(L2, u2m2));
    if (i >= 1) U0 = csub(U0, cmul(L1, u1m1));
    double2 U1 = cscale(e, c1[i]);
    if (i >= 1) U1 = csub(U1, cmul(L1, u2m1));
    const size_t o = (size_t)i * P.nb + l;
    P.l1[o] = L1;
    P.l2[o] = L2;
    P.iu0[o] = cinv(U0);
    P.u1[o] = U1;
    u0m2 = u0m1; u0m1 = U0;
    u1m2 = u1m1; u1m1 = U1;
    u2m2 = u2m1; u2m1 = cscale(e, c2[i]);
  }
}

// The solves are one thread per bin, so every row step is a dependent chain through the
// recurrence; the loads it needs are not.  Rows are processed in chunks of kPentaChunk whose loads
// are all issued before the chunk's arithmetic, so one memory latency is paid per chunk instead of
// per row (c2: 129 bins, i.e. 129 threads on the whole GPU — latency is all there is).
constexpr int kPentaChunk = 4;

// Solve L U x = b in place in `v` (column l of an [n][nb] array).
__device__ __noinline__ void penta_lu_solve(double2* __restrict__ v, int l, const PentaParams& P) {
  const int n = P.n, nb = P.nb;
  const double* __restrict__ c2 = P.band + 4 * n;
  const double2 e = P.el ? P.el[l] : make_double2(1.0, 0.0);
  double2 y1 = {0, 0}, y2 = {0, 0};
  for (int i0 = 0; i0 < n; i0 += kPentaChunk) {
    double2 vv[kPentaChunk], a1[kPentaChunk], a2[kPentaChunk];
#pragma unroll
    for (int k = 0; k < kPentaChunk; ++k)
      if (i0 + k < n) {
        const size_t o = (size_t)(i0 + k) * nb + l;
        vv[k] = v[o];
        a1[k] = P.l1[o];
        a2[k] = P.l2[o];
      }
#pragma unroll
    for (int k = 0; k < kPentaChunk; ++k)
      if (i0 + k < n) {
        double2 y = vv[k];
        y = csub(y, cmul(a1[k], y1));
        y = csub(y, cmul(a2[k], y2));
        v[(size_t)(i0 + k) * nb + l] = y;
        y2 = y1; y1 = y;
      }
  }
  double2 x1 = {0, 0}, x2 = {0, 0};
  for (int i1 = n - 1; i1 >= 0; i1 -= kPentaChunk) {
    double2 vv[kPentaChunk], b1[kPentaChunk], iu[kPentaChunk];
    double cc[kPentaChunk];
#pragma unroll
    for (int k = 0; k < kPentaChunk; ++k)
      if (i1 - k >= 0) {
        const int i = i1 - k;
        const size_t o = (size_t)i * nb + l;
        vv[k] = v[o];
        b1[k] = P.u1[o];
        iu[k] = P.iu0[o];
        cc[k] = c2[i];
      }
#pragma unroll
    for (int k = 0; k < kPentaChunk; ++k)
      if (i1 - k >= 0) {
        double2 x = vv[k];
        x = csub(x, cmul(b1[k], x1));
        x = csub(x, cscale(cmul(e, x2), cc[k]));
        x = cmul(x, iu[k]);
        v[(size_t)(i1 - k) * nb + l] = x;
        x2 = x1; x1 = x;
      }
  }
}

PD_DEV double2 ghost(const double2* v, int i, int l, const PentaParams& P) {
  const int n = P.n;
  if (i < 0 || i >= n) {
    if (!P.neumann) return make_double2(0.0, 0.0);
    i = i < 0 ? -i : 2 * (n - 1) - i;
  }
  return v[(size_t)i * P.nb + l];
}

// spec (in: ŝ, out: x), w1, w2 scratch [n][nb].  Refinement repeats (at most kPentaRefine times)
// until the correction is below 1e-15 of the iterate, per bin — the oracle's criterion (SURVEY
// §8(c) step 3.3) — or stops shrinking: a correction that is not at most half the previous one
// is rounding noise of the residual (the floor sits near cond·ε, above 1e-15 for c2), and further
// steps only stir it (measured: all six steps ran on c2, 0.71 ms of 0.81 per iteration).  One
// step suffices for c1/c2 (probe p10: 2.6e-7 → 1.8e-12); the condition number grows like m⁴, so
// longer lines (m = 8191: cond ≈ 1e14) need two or three.
constexpr int kPentaRefine = 6;
PD_DEV bool penta_refine_done(double cmax, double xmax, double& rprev) {
  const double r = cmax / xmax;
  const bool done = !(cmax > 1e-15 * xmax) || r > 0.5 * rprev;
  rprev = r;
  return done;
}

__global__ void k_penta_solve(double2* __restrict__ spec, double2* __restrict__ w1, double2* __restrict__ w2,
                              PentaParams P) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= P.nb) return;
  const int n = P.n, nb = P.nb;
  const double2 d = P.dl[l];
  const double2 e = P.el ? P.el[l] : make_double2(1.0, 0.0);
  constexpr int K = kPentaChunk;
  // x = (LU)^{-1} s
  for (int i0 = 0; i0 < n; i0 += K) {
    double2 t[K];
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (i0 + k < n) t[k] = spec[(size_t)(i0 + k) * nb + l];
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (i0 + k < n) w1[(size_t)(i0 + k) * nb + l] = t[k];
  }
  penta_lu_solve(w1, l, P);
  double rprev = INFINITY;
  for (int it = 0; it < P.refine; ++it) {
    // ρ = s - (d x + A x) into w2, A x in nested form from a sliding window of x values:
    // L x at i uses x_{i-1}, x_i, x_{i+1}; A x at i uses L x at i-1, i, i+1 (ghost rules of the BC)
    auto lap = [&](double2 xm, double2 xc, double2 xp) {
      return make_double2(((xm.x + xp.x) - 2.0 * xc.x) * P.inv_h2, ((xm.y + xp.y) - 2.0 * xc.y) * P.inv_h2);
    };
    // x at -1, 0, 1 (ghosts) and L x at -1, 0
    double2 xm1 = ghost(w1, -1, l, P), x0 = w1[l], xp1 = ghost(w1, 1, l, P);
    double2 lc = lap(xm1, x0, xp1);                          // L x at 0
    double2 lm;                                             // L x at -1 (ghost rule for L x)
    if (P.neumann) {
      const double2 x2 = ghost(w1, 2, l, P);
      lm = lap(x0, xp1, x2);                                 // L x_{-1} = L x_1 (even reflection)
    } else {
      lm = make_double2(0.0, 0.0);
    }
    double2 xa = x0, xb = xp1;                               // x_i, x_{i+1}
    for (int i0 = 0; i0 < n; i0 += K) {
      double2 xn[K], sv[K], xv[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int i = i0 + k;
        if (i < n) {
          xn[k] = ghost(w1, i + 2, l, P);                      // x_{i+2}
          sv[k] = spec[(size_t)i * nb + l];
          xv[k] = w1[(size_t)i * nb + l];
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int i = i0 + k;
        if (i < n) {
          // L x at i+1 (past the end: Neumann reflects, hinged ghost L = 0)
          double2 lp;
          if (i + 1 < n) lp = lap(xa, xb, xn[k]);
          else lp = P.neumann ? lm : make_double2(0.0, 0.0);
          const double2 ll = lap(lm, lc, lp);
          double2 Ax;
          if (P.kind == 0) Ax = ll;
          else Ax = make_double2(P.b2 * lc.x + P.e2 * ll.x, P.b2 * lc.y + P.e2 * ll.y);
          const double2 x = xv[k], s = sv[k];
          const double2 dx = cmul(d, x);
          const double2 eAx = P.el ? cmul(e, Ax) : Ax;
          w2[(size_t)i * nb + l] = make_double2(s.x - (dx.x + eAx.x), s.y - (dx.y + eAx.y));
          lm = lc; lc = lp;
          xa = xb; xb = xn[k];
        }
      }
    }
    penta_lu_solve(w2, l, P);
    double cmax = 0.0, xmax = 0.0;
    for (int i0 = 0; i0 < n; i0 += K) {
      double2 cv[K], xv[K];
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (i0 + k < n) {
          const size_t o = (size_t)(i0 + k) * nb + l;
          cv[k] = w2[o];
          xv[k] = w1[o];
        }
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (i0 + k < n) {
          const double2 x = cadd(xv[k], cv[k]);
          w1[(size_t)(i0 + k) * nb + l] = x;
          cmax = fmax(cmax, fmax(fabs(cv[k].x), fabs(cv[k].y)));
          xmax = fmax(xmax, fmax(fabs(x.x), fabs(x.y)));
        }
    }
    if (penta_refine_done(cmax, xmax, rprev)) break;
  }
  for (int i0 = 0; i0 < n; i0 += K) {
    double2 t[K];
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (i0 + k < n) t[k] = w1[(size_t)(i0 + k) * nb + l];
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (i0 + k < n) spec[(size_t)(i0 + k) * nb + l] = t[k];
  }
}

// ---- one CTA per bin (short lines, n ≤ kPentaCtaMaxN): the bin's factors, right-hand side and
// iterate live in shared memory; the nested residual, the update and the convergence test of
// every refinement step run row-parallel over the CTA, and the two LU sweeps (order-2 linear
// recurrences) run on warp 0 split into 32 row chunks:
//   pass 1  every lane runs its chunk three times side by side — the particular solution from a
//           zero entry state and the two homogeneous solutions from the unit entry states — which
//           gives the chunk's affine transfer map  S_out = p + S_in,1 · h + S_in,2 · g;
//   combine lane 0 chains the 32 maps (32 short steps instead of n) into every chunk's entry state;
//   pass 2  every lane re-runs its chunk from the exact entry state with the sequential sweep's
//           arithmetic, writing the result.
// The refinement that follows absorbs the (rounding-level) difference to the sequential sweep.
// Shared arrays are padded (index i + i/32) so the lanes' chunk-strided rows hit distinct banks.
// Same stop rule as k_penta_solve.
constexpr int kPentaCtaThreads = 256;
constexpr int kPentaCtaMaxN = 1920;
__host__ __device__ inline int pidx(int i) { return i + (i >> 5); }
inline size_t penta_cta_smem(int n) { return (size_t)7 * (pidx(n) + 1) * sizeof(double2); }

PD_DEV double2 cneg(double2 a) { return make_double2(-a.x, -a.y); }

// forward sweep y_i = (v_i - l1_i y_{i-1}) - l2_i y_{i-2} in place (warp 0)
PD_DEV void penta_fwd_warp(double2* v, const double2* L1, const double2* L2, int n, int lane, double2 (*mp)[6],
                           double2 (*st)[2]) {
  const int C = (n + 31) >> 5, a = lane * C, b = min(n, a + C);
  const double2 z = make_double2(0.0, 0.0), o = make_double2(1.0, 0.0);
  double2 p1 = z, p2 = z, h1 = o, h2 = z, g1 = z, g2 = o;     // (state_{i-1}, state_{i-2})
  for (int i = a; i < b; ++i) {
    const int q = pidx(i);
    const double2 l1 = L1[q], l2 = L2[q];
    const double2 yp = csub(csub(v[q], cmul(l1, p1)), cmul(l2, p2));
    const double2 yh = cneg(cadd(cmul(l1, h1), cmul(l2, h2)));
    const double2 yg = cneg(cadd(cmul(l1, g1), cmul(l2, g2)));
    p2 = p1; p1 = yp; h2 = h1; h1 = yh; g2 = g1; g1 = yg;
  }
  mp[lane][0] = p1; mp[lane][1] = p2; mp[lane][2] = h1; mp[lane][3] = h2; mp[lane][4] = g1; mp[lane][5] = g2;
  __syncwarp();
  if (lane == 0) {
    double2 s1 = z, s2 = z;                                   // y_{-1} = y_{-2} = 0
    for (int k = 0; k < 32; ++k) {
      st[k][0] = s1; st[k][1] = s2;
      const double2 o1 = cadd(mp[k][0], cadd(cmul(s1, mp[k][2]), cmul(s2, mp[k][4])));
      const double2 o2 = cadd(mp[k][1], cadd(cmul(s1, mp[k][3]), cmul(s2, mp[k][5])));
      s1 = o1; s2 = o2;
    }
  }
  __syncwarp();
  double2 y1 = st[lane][0], y2 = st[lane][1];
  for (int i = a; i < b; ++i) {
    const int q = pidx(i);
    double2 y = v[q];
    y = csub(y, cmul(L1[q], y1));
    y = csub(y, cmul(L2[q], y2));
    v[q] = y;
    y2 = y1; y1 = y;
  }
  __syncwarp();
}

// backward sweep x_i = ((y_i - u1_i x_{i+1}) - c2_i e x_{i+2}) / u0_i in place (warp 0)
PD_DEV void penta_bwd_warp(double2* v, const double2* U1, const double2* IU, const double* __restrict__ c2, double2 e,
                           int n, int lane, double2 (*mp)[6], double2 (*st)[2]) {
  const int C = (n + 31) >> 5, a = lane * C, b = min(n, a + C);
  const double2 z = make_double2(0.0, 0.0), o = make_double2(1.0, 0.0);
  double2 p1 = z, p2 = z, h1 = o, h2 = z, g1 = z, g2 = o;     // (state_{i+1}, state_{i+2})
  for (int i = b - 1; i >= a; --i) {
    const int q = pidx(i);
    const double2 u1 = U1[q], iu = IU[q];
    const double c = __ldg(c2 + i);
    const double2 xp = cmul(csub(csub(v[q], cmul(u1, p1)), cscale(cmul(e, p2), c)), iu);
    const double2 xh = cmul(cneg(cadd(cmul(u1, h1), cscale(cmul(e, h2), c))), iu);
    const double2 xg = cmul(cneg(cadd(cmul(u1, g1), cscale(cmul(e, g2), c))), iu);
    p2 = p1; p1 = xp; h2 = h1; h1 = xh; g2 = g1; g1 = xg;
  }
  mp[lane][0] = p1; mp[lane][1] = p2; mp[lane][2] = h1; mp[lane][3] = h2; mp[lane][4] = g1; mp[lane][5] = g2;
  __syncwarp();
  if (lane == 0) {
    double2 s1 = z, s2 = z;                                   // x_n = x_{n+1} = 0
    for (int k = 31; k >= 0; --k) {
      st[k][0] = s1; st[k][1] = s2;
      const double2 o1 = cadd(mp[k][0], cadd(cmul(s1, mp[k][2]), cmul(s2, mp[k][4])));
      const double2 o2 = cadd(mp[k][1], cadd(cmul(s1, mp[k][3]), cmul(s2, mp[k][5])));
      s1 = o1; s2 = o2;
    }
  }
  __syncwarp();
  double2 x1 = st[lane][0], x2 = st[lane][1];
  for (int i = b - 1; i >= a; --i) {
    const int q = pidx(i);
    double2 x = v[q];
    x = csub(x, cmul(U1[q], x1));
    x = csub(x, cscale(cmul(e, x2), __ldg(c2 + i)));
    x = cmul(x, IU[q]);
    v[q] = x;
    x2 = x1; x1 = x;
  }
  __syncwarp();
}

PD_DEV double2 ghost_s(const double2* v, int i, int n, int neumann) {
  if (i < 0 || i >= n) {
    if (!neumann) return make_double2(0.0, 0.0);
    i = i < 0 ? -i : 2 * (n - 1) - i;
  }
  return v[pidx(i)];
}

__global__ void __launch_bounds__(kPentaCtaThreads)
k_penta_solve_cta(double2* __restrict__ spec, PentaParams P) {
  extern __shared__ double2 ps[];
  const int l = blockIdx.x, n = P.n, nb = P.nb, tid = threadIdx.x, lane = tid & 31;
  const int ld = pidx(n) + 1;
  double2* s_ = ps;                 // right-hand side ŝ
  double2* x_ = ps + ld;            // iterate
  double2* w_ = ps + 2 * ld;        // residual / correction
  double2* L1 = ps + 3 * ld;
  double2* L2 = ps + 4 * ld;
  double2* U1 = ps + 5 * ld;
  double2* IU = ps + 6 * ld;
  __shared__ double2 mp[32][6], st[32][2];
  __shared__ double red[2][kPentaCtaThreads / 32];
  __shared__ int stop;
  for (int i = tid; i < n; i += kPentaCtaThreads) {
    const size_t o = (size_t)i * nb + l;
    const int q = pidx(i);
    const double2 v = spec[o];
    s_[q] = v;
    x_[q] = v;
    L1[q] = P.l1[o];
    L2[q] = P.l2[o];
    U1[q] = P.u1[o];
    IU[q] = P.iu0[o];
  }
  __syncthreads();
  const double2 d = P.dl[l];
  const double2 e = P.el ? P.el[l] : make_double2(1.0, 0.0);
  const double* __restrict__ c2 = P.band + 4 * n;
  auto lu = [&](double2* v) {
    if (tid < 32) {
      penta_fwd_warp(v, L1, L2, n, lane, mp, st);
      penta_bwd_warp(v, U1, IU, c2, e, n, lane, mp, st);
    }
    __syncthreads();
  };
  auto lapx = [&](int i) {                            // L x at i (x with the BC's ghost rule)
    const double2 xm = ghost_s(x_, i - 1, n, P.neumann), xc = ghost_s(x_, i, n, P.neumann),
                  xp = ghost_s(x_, i + 1, n, P.neumann);
    return make_double2(((xm.x + xp.x) - 2.0 * xc.x) * P.inv_h2, ((xm.y + xp.y) - 2.0 * xc.y) * P.inv_h2);
  };
  auto lapg = [&](int i) {                            // L x at a possibly-ghost position
    if (i < 0 || i >= n) {
      if (!P.neumann) return make_double2(0.0, 0.0);
      i = i < 0 ? -i : 2 * (n - 1) - i;
    }
    return lapx(i);
  };
  lu(x_);
  double rprev = INFINITY;                            // thread 0's stagnation state
  for (int it = 0; it < P.refine; ++it) {
    // ρ = s - (d x + A x), A x nested (R#15): ((L_{i-1} + L_{i+1}) - 2 L_i) / h², row-parallel
    for (int i = tid; i < n; i += kPentaCtaThreads) {
      const int q = pidx(i);
      const double2 lc = lapx(i), lm = lapg(i - 1), lp = lapg(i + 1);
      const double2 ll = make_double2(((lm.x + lp.x) - 2.0 * lc.x) * P.inv_h2, ((lm.y + lp.y) - 2.0 * lc.y) * P.inv_h2);
      double2 Ax;
      if (P.kind == 0) Ax = ll;
      else Ax = make_double2(P.b2 * lc.x + P.e2 * ll.x, P.b2 * lc.y + P.e2 * ll.y);
      const double2 x = x_[q], sv = s_[q];
      const double2 dx = cmul(d, x);
      const double2 eAx = P.el ? cmul(e, Ax) : Ax;
      w_[q] = make_double2(sv.x - (dx.x + eAx.x), sv.y - (dx.y + eAx.y));
    }
    __syncthreads();
    lu(w_);
    double cmax = 0.0, xmax = 0.0;
    for (int i = tid; i < n; i += kPentaCtaThreads) {
      const int q = pidx(i);
      const double2 c = w_[q];
      const double2 x = cadd(x_[q], c);
      x_[q] = x;
      cmax = fmax(cmax, fmax(fabs(c.x), fabs(c.y)));
      xmax = fmax(xmax, fmax(fabs(x.x), fabs(x.y)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
      xmax = fmax(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
    }
    if ((tid & 31) == 0) {
      red[0][tid >> 5] = cmax;
      red[1][tid >> 5] = xmax;
    }
    __syncthreads();
    if (tid == 0) {
      double c = 0.0, x = 0.0;
      for (int w = 0; w < kPentaCtaThreads / 32; ++w) {
        c = fmax(c, red[0][w]);
        x = fmax(x, red[1][w]);
      }
      stop = penta_refine_done(c, x, rprev);
    }
    __syncthreads();
    if (stop) break;
  }
  for (int i = tid; i < n; i += kPentaCtaThreads) spec[(size_t)i * nb + l] = x_[pidx(i)];
}

}  // namespace pd
