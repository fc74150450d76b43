// k_misc.cuh — defect-correction update U ← U + ω δ (R#9 damping), initial iterates, scalars.
#pragma once
#include "common.cuh"

namespace pd {

PD_DEV double stats_omega(const DevStats* st, int damped, double omega_cap, double tau) {
  if (!damped) return 1.0;
  const double dmax = __longlong_as_double((long long)st->dmax_bits);
  return dmax > 0.0 ? fmin(omega_cap, tau / dmax) : omega_cap;
}

// U += ω δ over n doubles; ‖U‖∞ reduced into st->umax_bits.  Vectorised by double2 when aligned.
// Usrc == U: in place.  Otherwise U = Usrc + ω δ (the pipelined solve's last update lands in the
// caller's buffer from the alternate one).
__global__ void __launch_bounds__(256)
k_update(double* U, const double* delta, size_t n, DevStats* st, int damped, double omega_cap, double tau,
         const double* Usrc = nullptr, int want_dmax = 0) {
  if (!Usrc) Usrc = U;
  const double w = stats_omega(st, damped, omega_cap, tau);
  if (blockIdx.x == 0 && threadIdx.x == 0) st->omega = w;
  // ‖U‖∞ as a max over |u| bit patterns: NaN sorts above +inf, so a non-finite iterate always
  // reaches the host check (the ‖δ‖∞ epilogues of the line passes do not propagate NaN)
  unsigned long long lbits = 0ull;
  const unsigned long long absmask = 0x7fffffffffffffffull;
  if ((reinterpret_cast<uintptr_t>(U) | reinterpret_cast<uintptr_t>(Usrc) | reinterpret_cast<uintptr_t>(delta)) & 15) {
    // a slice range of an odd-sized slab (chunked multi-rank schedule): scalar path
    unsigned long long db = 0ull;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const double u = Usrc[i] + w * delta[i];
      U[i] = u;
      lbits = max(lbits, (unsigned long long)__double_as_longlong(u) & absmask);
      if (want_dmax) db = max(db, (unsigned long long)__double_as_longlong(delta[i]) & absmask);
    }
    lbits = warp_max_u64(lbits);
    if ((threadIdx.x & 31) == 0 && lbits) atomicMax(&st->umax_bits, lbits);
    if (want_dmax) {
      db = warp_max_u64(db);
      if ((threadIdx.x & 31) == 0 && db) atomicMax(&st->dmax_bits, db);
    }
    return;
  }
  const size_t n2 = n / 2;
  double2* U2 = reinterpret_cast<double2*>(U);
  const double2* S2 = reinterpret_cast<const double2*>(Usrc);
  const double2* D2 = reinterpret_cast<const double2*>(delta);
  // want_dmax (ω = 1 only): ‖δ‖∞ here, as a bit-pattern max like ‖U‖∞, instead of in the last line pass
  unsigned long long dbits = 0ull;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 u = S2[i];
    const double2 d = __ldg(D2 + i);
    u.x += w * d.x;
    u.y += w * d.y;
    U2[i] = u;
    const unsigned long long bx = (unsigned long long)__double_as_longlong(u.x) & absmask;
    const unsigned long long by = (unsigned long long)__double_as_longlong(u.y) & absmask;
    lbits = max(lbits, max(bx, by));
    if (want_dmax)
      dbits = max(dbits, max((unsigned long long)__double_as_longlong(d.x) & absmask,
                             (unsigned long long)__double_as_longlong(d.y) & absmask));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const double u = Usrc[n - 1] + w * delta[n - 1];
    U[n - 1] = u;
    lbits = max(lbits, (unsigned long long)__double_as_longlong(u) & absmask);
    if (want_dmax) dbits = max(dbits, (unsigned long long)__double_as_longlong(delta[n - 1]) & absmask);
  }
  lbits = warp_max_u64(lbits);
  if ((threadIdx.x & 31) == 0 && lbits) atomicMax(&st->umax_bits, lbits);
  if (want_dmax) {
    dbits = warp_max_u64(dbits);
    if ((threadIdx.x & 31) == 0 && dbits) atomicMax(&st->dmax_bits, dbits);
  }
}

// U⁰: broadcast u0 to every time slice, or zero (R#5).
__global__ void k_init_iterate(double* __restrict__ U, const double* __restrict__ u0, size_t ns,
                               size_t total, int zero) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x)
    U[i] = zero ? 0.0 : __ldg(u0 + i % ns);
}

__global__ void k_reset_stats(DevStats* st) {
  st->dmax_bits = 0ull;
  st->umax_bits = 0ull;
  st->omega = 1.0;      // the fused x-inverse + update pass (linear kinds) applies ω = 1
}

__global__ void k_set_jbar(DevStats* st, double jbar) { st->jbar = jbar; }

// dst[a·d0 + b·d1 + c] = src[a·s0 + b·s1 + c] for a < n0, b < n1, c < n2 — the pack / unpack of
// the row-slab <-> column-slab transposes of a multi-rank run (one CTA per (a, b) row, grid-stride).
__global__ void __launch_bounds__(256)
k_copy3d(const double* __restrict__ src, double* __restrict__ dst, int64_t n0, int64_t n1, int64_t n2,
         int64_t s0, int64_t s1, int64_t d0, int64_t d1) {
  for (int64_t row = blockIdx.x; row < n0 * n1; row += gridDim.x) {
    const int64_t a = row / n1, b = row - a * n1;
    const double* s = src + a * s0 + b * s1;
    double* d = dst + a * d0 + b * d1;
    for (int64_t c = threadIdx.x; c < n2; c += blockDim.x) d[c] = __ldg(s + c);
  }
}

}  // namespace pd
