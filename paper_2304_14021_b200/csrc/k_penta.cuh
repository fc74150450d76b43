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

// Solve L U x = b in place in `v` (column l of an [n][nb] array).
PD_DEV void penta_lu_solve(double2* v, int l, const PentaParams& P) {
  const int n = P.n, nb = P.nb;
  const double* c2 = P.band + 4 * n;
  const double2 e = P.el ? P.el[l] : make_double2(1.0, 0.0);
  double2 y1 = {0, 0}, y2 = {0, 0};
  for (int i = 0; i < n; ++i) {
    const size_t o = (size_t)i * nb + l;
    double2 y = v[o];
    y = csub(y, cmul(P.l1[o], y1));
    y = csub(y, cmul(P.l2[o], y2));
    v[o] = y;
    y2 = y1; y1 = y;
  }
  double2 x1 = {0, 0}, x2 = {0, 0};
  for (int i = n - 1; i >= 0; --i) {
    const size_t o = (size_t)i * nb + l;
    double2 x = v[o];
    x = csub(x, cmul(P.u1[o], x1));
    x = csub(x, cscale(cmul(e, x2), c2[i]));
    x = cmul(x, P.iu0[o]);
    v[o] = x;
    x2 = x1; x1 = x;
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
// §8(c) step 3.3).  One step suffices for c1/c2 (probe p10: 2.6e-7 → 1.8e-12); the condition
// number grows like m⁴, so longer lines (m = 8191: cond ≈ 1e14) need two or three.
constexpr int kPentaRefine = 6;

__global__ void k_penta_solve(double2* spec, double2* w1, double2* w2, PentaParams P) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= P.nb) return;
  const int n = P.n, nb = P.nb;
  const double2 d = P.dl[l];
  const double2 e = P.el ? P.el[l] : make_double2(1.0, 0.0);
  // x = (LU)^{-1} s
  for (int i = 0; i < n; ++i) w1[(size_t)i * nb + l] = spec[(size_t)i * nb + l];
  penta_lu_solve(w1, l, P);
  for (int it = 0; it < kPentaRefine; ++it) {
    // w2 = L x (nested Laplacian with the BC's ghost rule)
    for (int i = 0; i < n; ++i) {
      const double2 xm = ghost(w1, i - 1, l, P), xc = w1[(size_t)i * nb + l], xp = ghost(w1, i + 1, l, P);
      w2[(size_t)i * nb + l] = make_double2(((xm.x + xp.x) - 2.0 * xc.x) * P.inv_h2,
                                            ((xm.y + xp.y) - 2.0 * xc.y) * P.inv_h2);
    }
    // ρ = s - (d x + A x), written over w2 with a sliding window of L x values
    double2 lm = ghost(w2, -1, l, P);
    double2 lc = w2[l];
    for (int i = 0; i < n; ++i) {
      // L x at i+1; past the end the ghost is L x_{n-2} (Neumann, = lm here) or 0 (hinged)
      const double2 lp = i + 1 < n ? w2[(size_t)(i + 1) * nb + l]
                                   : (P.neumann ? lm : make_double2(0.0, 0.0));
      const double2 ll = make_double2(((lm.x + lp.x) - 2.0 * lc.x) * P.inv_h2,
                                      ((lm.y + lp.y) - 2.0 * lc.y) * P.inv_h2);
      double2 Ax;
      if (P.kind == 0) Ax = ll;
      else Ax = make_double2(P.b2 * lc.x + P.e2 * ll.x, P.b2 * lc.y + P.e2 * ll.y);
      const size_t o = (size_t)i * nb + l;
      const double2 x = w1[o], s = spec[o];
      const double2 dx = cmul(d, x);
      const double2 eAx = P.el ? cmul(e, Ax) : Ax;
      w2[o] = make_double2(s.x - (dx.x + eAx.x), s.y - (dx.y + eAx.y));
      lm = lc; lc = lp;
    }
    penta_lu_solve(w2, l, P);
    double cmax = 0.0, xmax = 0.0;
    for (int i = 0; i < n; ++i) {
      const size_t o = (size_t)i * nb + l;
      const double2 c = w2[o];
      const double2 x = cadd(w1[o], c);
      w1[o] = x;
      cmax = fmax(cmax, fmax(fabs(c.x), fabs(c.y)));
      xmax = fmax(xmax, fmax(fabs(x.x), fabs(x.y)));
    }
    if (!(cmax > 1e-15 * xmax)) break;
  }
  for (int i = 0; i < n; ++i) {
    const size_t o = (size_t)i * nb + l;
    spec[o] = w1[o];
  }
}

}  // namespace pd
