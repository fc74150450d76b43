// common.cuh — complex helpers, reductions and small utilities shared by the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define PD_DEV __device__ __forceinline__

namespace pd {

PD_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
PD_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
PD_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
PD_DEV double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
PD_DEV double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

// 1 / z
PD_DEV double2 cinv(double2 z) {
  const double q = 1.0 / (z.x * z.x + z.y * z.y);
  return make_double2(z.x * q, -z.y * q);
}

// 1 / z without a division: hardware reciprocal estimate of |z|² refined by two Newton steps
// (≤ 1 ulp from the correctly rounded value; no branch, |z|² is a normal positive number here).
PD_DEV double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
PD_DEV double2 cinv_fast(double2 z) {
  const double q = rcp_fast(z.x * z.x + z.y * z.y);
  return make_double2(z.x * q, -z.y * q);
}

// Device-resident per-iteration scalars.  |x| of a finite double orders like its bit pattern, so a
// max-abs reduction is an integer atomicMax on the bits (deterministic; NaN sorts above +inf).
struct DevStats {
  unsigned long long dmax_bits;   // ‖δ‖∞ of the last preconditioner application
  unsigned long long umax_bits;   // ‖U‖∞ after the update
  double jbar;                    // J̄ = mean(3U² - 1) (CH)
  double omega;                   // damping applied by the update
};

PD_DEV unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

PD_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Running max of |v| for the ‖δ‖∞ epilogues: a compare + select (fmax's NaN rules cost ~4x the
// instructions).  A NaN is not propagated here; it reaches U through the update, whose ‖U‖∞
// reduction (bit-pattern max, NaN sorts above +inf) and the host isfinite check catch it.
PD_DEV double amax_acc(double m, double v) {
  const double a = fabs(v);
  return a > m ? a : m;
}

// Block-wide max of |v| folded into *dst with one atomic per warp.
PD_DEV void warp_atomic_max_abs(unsigned long long* dst, double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v));
  b = warp_max_u64(b);
  if ((threadIdx.x & 31) == 0 && b) atomicMax(dst, b);
}

PD_DEV int bitrev(int v, int bits) { return bits ? (int)(__brev((unsigned)v) >> (32 - bits)) : 0; }

// SMEM index padding: one 16-byte slot per 16 complex values keeps strided radix passes
// conflict-free (stride-16 lanes land on consecutive 16-byte bank groups).
PD_DEV int pad16(int p) { return p + (p >> 4); }
__host__ __device__ constexpr int padded16(int n) { return n + (n >> 4) + 1; }

}  // namespace pd

namespace pd {

// ---- cp.async (LDGSTS): global -> shared without register staging; many copies in flight
PD_DEV void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
PD_DEV void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
PD_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
PD_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
template <int N>
PD_DEV void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Double-index padding of a line buffer: two doubles (one complex slot) per 32 doubles, so that the
// complex view of the same buffer is exactly pad16() (2·pad16(n) == dpad(2n)).
PD_DEV int dpad(int j) { return j + 2 * (j >> 5); }
__host__ __device__ constexpr int dpadded(int m) { return ((m + 2 * (m >> 5) + 2) + 1) & ~1; }

}  // namespace pd
