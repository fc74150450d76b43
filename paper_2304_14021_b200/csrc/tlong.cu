// tlong.cu — launch wrappers of the long-window time pass (k_tlong.cuh), one instantiation per
// transform length 32·E of each four-step factor.  paradiag.cu sees only tlong.h.
#define PD_TLONG_KERNELS
#include "tlong.h"
#include "k_tmix.cuh"

#include <algorithm>

namespace pd {

namespace {

template <int E>
cudaError_t attrs_e() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_tl_a_fwd<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTlSmem))) return e;
  if ((e = cudaFuncSetAttribute(k_tl_b_fwd<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTlSmem))) return e;
  if ((e = cudaFuncSetAttribute(k_tl_b_inv<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTlSmem))) return e;
  return cudaFuncSetAttribute(k_tl_a_inv<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTlSmem);
}

// CTAs of a pass over transform length L = 32·E: (N / L) / (32 / E) groups × chunks
unsigned grid_of(int L, const TlongParams& Q) {
  const int64_t groups = (int64_t)(Q.N / L) / (1024 / L);
  return (unsigned)(groups * Q.nch);
}

template <int E>
void launch_e(int stage, const void* in, void* out, const TlongParams& Q, cudaStream_t s) {
  constexpr int L = 32 * E;
  const unsigned grid = grid_of(L, Q);
  switch (stage) {
    case 0: k_tl_a_fwd<E><<<grid, kTlThreads, kTlSmem, s>>>(static_cast<const double*>(in), static_cast<double2*>(out), Q); break;
    case 1: k_tl_b_fwd<E><<<grid, kTlThreads, kTlSmem, s>>>(static_cast<const double2*>(in), static_cast<double2*>(out), Q); break;
    case 3: k_tl_b_inv<E><<<grid, kTlThreads, kTlSmem, s>>>(static_cast<const double2*>(in), static_cast<double2*>(out), Q); break;
    case 4: k_tl_a_inv<E><<<grid, kTlThreads, kTlSmem, s>>>(static_cast<const double2*>(in), static_cast<double*>(out), Q); break;
    default: break;
  }
}

}  // namespace

void tlong_split(int log2N, int* log2N1, int* log2N2) {
  // N2 = 1024 whenever N1 = N / 1024 ≥ 32 (the fused pass B needs N2 = 1024), else balanced
  if (log2N >= 15) {
    *log2N2 = 10;
  } else {
    *log2N2 = log2N / 2;
  }
  *log2N1 = log2N - *log2N2;
}

// power of two: k_tl_b_fused (N2 = 1024); mixed radix: k_mx_b_fused (any split, N2 ≤ kMixMaxL)
bool tlong_fusable(const TlongParams& Q) { return Q.mixed ? Q.N1 >= 2 : (Q.N2 == 1024 && Q.N1 >= 32); }

bool mixed_split(int N, int* N1, int* N2, int8_t* plan1, int* ns1, int8_t* plan2, int* ns2) {
  auto smooth = [](int v) {
    while (v % 2 == 0) v /= 2;
    while (v % 5 == 0) v /= 5;
    return v == 1;
  };
  if (N < 64 || !smooth(N)) return false;
  int best = 0;
  for (int a = 8; a <= kMixMaxL && (int64_t)a * a <= N; ++a)          // largest N1 ≤ √N with both factors ≤ kMixMaxL
    if (N % a == 0 && smooth(a) && N / a <= kMixMaxL) best = a;
  if (!best) return false;
  *N1 = best;
  *N2 = N / best;
  auto plan = [](int L, int8_t* p, int* n) {
    *n = 0;
    for (int r : {8, 4, 2}) while (L % r == 0) { p[(*n)++] = (int8_t)r; L /= r; }
    while (L % 5 == 0) { p[(*n)++] = 5; L /= 5; }
  };
  plan(*N1, plan1, ns1);
  plan(*N2, plan2, ns2);
  return true;
}

cudaError_t tlong_attrs() {
  cudaError_t e;
  if ((e = attrs_e<1>()) || (e = attrs_e<2>()) || (e = attrs_e<4>()) || (e = attrs_e<8>()) || (e = attrs_e<16>()) ||
      (e = attrs_e<32>()))
    return e;
  if ((e = cudaFuncSetAttribute(k_tl_b_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFbSmem)))
    return e;
#define PD_MXA(K, B)                                                                              \
  if ((e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(B)))) return e;
  PD_MXA(k_mx_a_fwd<8>, mx_pass_smem<8>()) PD_MXA(k_mx_a_inv<8>, mx_pass_smem<8>())
  PD_MXA(k_mx_b_fwd<8>, mx_pass_smem<8>()) PD_MXA(k_mx_b_inv<8>, mx_pass_smem<8>())
  PD_MXA(k_mx_a_fwd<4>, mx_pass_smem<4>()) PD_MXA(k_mx_a_inv<4>, mx_pass_smem<4>())
  PD_MXA(k_mx_b_fwd<4>, mx_pass_smem<4>()) PD_MXA(k_mx_b_inv<4>, mx_pass_smem<4>())
  PD_MXA((k_mx_b_fused<true, 4>), mx_fused_smem<4>()) PD_MXA((k_mx_b_fused<false, 4>), mx_fused_smem<4>())
  PD_MXA((k_mx_b_fused<true, 2>), mx_fused_smem<2>()) PD_MXA((k_mx_b_fused<false, 2>), mx_fused_smem<2>())
#undef PD_MXA
  return cudaFuncSetAttribute(k_tl_b_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFbSmem);
}

bool tlong_launch(int stage, const void* in, void* out, const TlongParams& Q, cudaStream_t s) {
  if (stage == 5) {                                     // fused B: Y in place (`out`)
    if (!tlong_fusable(Q)) return false;
    if (Q.mixed) {
      const int mp = Q.mxp / 2;                          // pairs per group
      const int64_t nch4 = (Q.P + mp - 1) / mp;
      const unsigned grid = (unsigned)(nch4 * ((Q.N1 - 1) / 2 + 1));
      double2* y = static_cast<double2*>(out);
      const bool plain = !Q.T.el && !Q.T.l3;
      if (mp == 2) {
        if (plain) k_mx_b_fused<true, 2><<<grid, 256, mx_fused_smem<2>(), s>>>(y, Q);
        else k_mx_b_fused<false, 2><<<grid, 256, mx_fused_smem<2>(), s>>>(y, Q);
      } else {
        if (plain) k_mx_b_fused<true, 4><<<grid, 512, mx_fused_smem<4>(), s>>>(y, Q);
        else k_mx_b_fused<false, 4><<<grid, 512, mx_fused_smem<4>(), s>>>(y, Q);
      }
      return true;
    }
    const int64_t nch4 = (Q.P + kFbPairs - 1) / kFbPairs;
    const unsigned grid = (unsigned)(nch4 * (Q.N1 / 2));
    if (!Q.T.el && !Q.T.l3) k_tl_b_fused<true><<<grid, kFbThreads, kFbSmem, s>>>(static_cast<double2*>(out), Q);
    else k_tl_b_fused<false><<<grid, kFbThreads, kFbSmem, s>>>(static_cast<double2*>(out), Q);
    return true;
  }
  if (Q.mixed && stage != 2) {                          // mixed radix (k_tmix.cuh): one transform per CTA
    const int np = Q.mxp;                               // pencil pairs per CTA: 8 or 4
    const unsigned grid = (unsigned)(((Q.P + np - 1) / np) * ((stage == 0 || stage == 4) ? Q.N2 : Q.N1));
    const size_t sm = np == 4 ? mx_pass_smem<4>() : mx_pass_smem<8>();
    const unsigned nt = (unsigned)(np * kMxWpp * 32);
#define PD_MX(NP)                                                                                          \
    switch (stage) {                                                                                       \
      case 0: k_mx_a_fwd<NP><<<grid, nt, sm, s>>>(static_cast<const double*>(in), static_cast<double2*>(out), Q); break; \
      case 1: k_mx_b_fwd<NP><<<grid, nt, sm, s>>>(static_cast<const double2*>(in), static_cast<double2*>(out), Q); break; \
      case 3: k_mx_b_inv<NP><<<grid, nt, sm, s>>>(static_cast<const double2*>(in), static_cast<double2*>(out), Q); break; \
      case 4: k_mx_a_inv<NP><<<grid, nt, sm, s>>>(static_cast<const double2*>(in), static_cast<double*>(out), Q); break; \
      default: return false;                                                                               \
    }
    if (np == 4) { PD_MX(4) } else { PD_MX(8) }
#undef PD_MX
    return true;
  }
  if (stage == 2) {
    const int64_t total = (int64_t)(Q.N / 2 + 1) * Q.P;
    const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 8);
    k_tl_divide<<<grid, 256, 0, s>>>(static_cast<double2*>(out), Q);
    return true;
  }
  const int L = (stage == 0 || stage == 4) ? Q.N1 : Q.N2;
  switch (L) {
    case 32: launch_e<1>(stage, in, out, Q, s); return true;
    case 64: launch_e<2>(stage, in, out, Q, s); return true;
    case 128: launch_e<4>(stage, in, out, Q, s); return true;
    case 256: launch_e<8>(stage, in, out, Q, s); return true;
    case 512: launch_e<16>(stage, in, out, Q, s); return true;
    case 1024: launch_e<32>(stage, in, out, Q, s); return true;
    default: return false;
  }
}

}  // namespace pd
