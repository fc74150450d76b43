// fast_launch.cuh — launch wrappers of the register-FFT passes (k_dtt.cuh line transforms,
// k_fast.cuh time pass), one instantiation per E = transform length / 32 in its own translation
// unit (fast_e<E>.cu) so the library builds in parallel.  paradiag.cu sees only the declarations.
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>

#include <algorithm>

#include "k_dtt.cuh"
#include "k_dttp.cuh"
#include "k_fast.cuh"

namespace pd {

constexpr int kFastTimeWarps = 4;  // k_time2d_v2: warps per CTA
constexpr int kFastRowWarps = 4;   // k_rows3: warps per CTA (independent)
// column kernels: warps per CTA (C = warps·32/E adjacent columns per tile)
constexpr int fast_col_warps(int E) { return E == 1 ? 2 : E == 2 ? 4 : 8; }

struct FastLaunch {
  cudaStream_t stream;
  int nt;                 // time slices
  int nx;                 // points per row (square grids)
  int64_t ns;             // points per slice
  const double2* trig2;   // k_dtt.cuh split table
  const double2* trig2p;  // k_dttp.cuh split table (M = 2048 only)
  int dtt_ver;            // 4 = k_dttp.cuh (M = 2048, opt-in), otherwise k_dtt.cuh
};

template <int E>
cudaError_t fast_attrs();
template <int E>
void fast_line(int neumann, int axis, const double* in, double* out, const LineParams& L, const FastLaunch& F);
// y pass between the natural layout and the column-major workspace (k_cols_cm): dir 0 natural -> wt,
// dir 1 wt -> natural; lp = wt line pitch
template <int E>
void fast_cols_cm(int neumann, int dir, const double* in, double* out, const LineParams& L, const FastLaunch& F,
                  int64_t lp);
template <int E>
void fast_time(const double* in, double* out, const TimeParams& T, const FastLaunch& F);
// y⁻¹ pass with TMA box stores into the padded workspace that tmo describes (k_cols_tma_inv;
// M = 2048 only).  Returns false when this E has none.
template <int E>
bool fast_cols_tma_inv(int neumann, const double* in, const LineParams& L, const FastLaunch& F, int64_t lp,
                       const CUtensorMap* tmo);
// TMA-staged three-stage time pass (k_time2d_v4), in place on the buffer tmap describes: [N_t][ps]
// with ps = N_s rounded up to even, box {16, min(N_t, 256)}.  Returns false when this E has none.
template <int E>
bool fast_time_tma(double* buf, const TimeParams& T, const FastLaunch& F, const CUtensorMap* tmap);

#ifdef PD_FAST_DEFINE
template <int E>
constexpr size_t fast_time4_smem() {
  constexpr size_t S = 2 * (32 / E) * 4, tile = (size_t)S * 32 * E * 8, scr = (size_t)4 * kWarpBufD * 8;
  return 3 * (((tile > scr ? tile : scr) + 1023) & ~(size_t)1023) + (size_t)2 * 32 * E * 16 + 3 * 8;
}
inline size_t fast_time_smem(int E, int nw = kFastTimeWarps) {
  const size_t S = 2 * (32 / E) * nw, tile = (size_t)32 * E * (S + 1);
  return std::max(tile, (size_t)nw * kWarpBufD) * sizeof(double);
}
constexpr int kPairsPerRowCta = 2;
inline size_t dttp_rows_smem() { return (size_t)kPairsPerRowCta * DttPair<1>::BUF * sizeof(double); }
inline size_t dttp_cols_smem() { return (size_t)8 * DttPair<1>::BUF * sizeof(double); }
template <int E>
size_t dtt3_rows_smem() { return (size_t)kFastRowWarps * Dtt3<1, E>::BUF * sizeof(double); }
// k_rows3 with bulk row loads (BK = 1): the per-warp mbarriers follow the line buffers
template <int E>
size_t dtt3_rows_bulk_smem() { return dtt3_rows_smem<E>() + kFastRowWarps * 8; }
template <int E>
size_t dtt3_cols_smem() { return (size_t)fast_col_warps(E) * Dtt3<1, E>::BUF * sizeof(double); }

#define PD_ATTR(k, b)                                                                            \
  do {                                                                                           \
    cudaError_t e_ = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(b)); \
    if (e_ != cudaSuccess) return e_;                                                            \
  } while (0)

template <int E>
cudaError_t fast_attrs() {
  if constexpr (E <= 16 && fast_time4_smem<E>() <= 227 * 1024) {
    PD_ATTR((k_time2d_v4<E, 0>), fast_time4_smem<E>());
    PD_ATTR((k_time2d_v4<E, 1>), fast_time4_smem<E>());
    PD_ATTR((k_time2d_v4<E, 2>), fast_time4_smem<E>());
    PD_ATTR((k_time2d_v4<E, 3>), fast_time4_smem<E>());
  }
  PD_ATTR((k_time2d_v2<E, kFastTimeWarps, 0>), fast_time_smem(E));
  PD_ATTR((k_time2d_v2<E, kFastTimeWarps, 1>), fast_time_smem(E));
  PD_ATTR((k_time2d_v2<E, kFastTimeWarps, 2>), fast_time_smem(E));
  PD_ATTR((k_time2d_v2<E, kFastTimeWarps, 3>), fast_time_smem(E));
  if (fast_time_smem(E, 8) <= 227 * 1024) PD_ATTR((k_time2d_v2<E, 8>), fast_time_smem(E, 8));
  if constexpr (E == 32) {    // the table variant of the row pass (A/B, tune 2^24)
    PD_ATTR((k_rows3<1, E, kFastRowWarps, 0, 0>), dtt3_rows_smem<E>());
    PD_ATTR((k_rows3<0, E, kFastRowWarps, 0, 0>), dtt3_rows_smem<E>());
    PD_ATTR((k_rows3<1, E, kFastRowWarps, 0, kDttCT, 1>), dtt3_rows_bulk_smem<E>());
  }
  PD_ATTR((k_rows3<1, E, kFastRowWarps, 0>), dtt3_rows_smem<E>() + 100 * 1024);
  PD_ATTR((k_rows3<0, E, kFastRowWarps, 0>), dtt3_rows_smem<E>() + 100 * 1024);
  PD_ATTR((k_rows3<1, E, kFastRowWarps, 1>), dtt3_rows_smem<E>() + 100 * 1024);
  PD_ATTR((k_rows3<0, E, kFastRowWarps, 1>), dtt3_rows_smem<E>() + 100 * 1024);
  PD_ATTR((k_rows3<1, E, kFastRowWarps, 2>), dtt3_rows_smem<E>() + 100 * 1024);
  PD_ATTR((k_rows3<0, E, kFastRowWarps, 2>), dtt3_rows_smem<E>() + 100 * 1024);
  PD_ATTR((k_rows3<1, E, kFastRowWarps, 3>), dtt3_rows_smem<E>() + 100 * 1024);
  PD_ATTR((k_rows3<0, E, kFastRowWarps, 3>), dtt3_rows_smem<E>() + 100 * 1024);
  if constexpr (E == 32) {   // (A/B) PARADIAG_CARVE: preferred shared-memory carve-out (percent) of the cp.async line passes
    if (const char* cv = getenv("PARADIAG_CARVE")) {
      const int pc = atoi(cv);
      cudaFuncSetAttribute(k_cols_cm<1, E, fast_col_warps(E), 0>, cudaFuncAttributePreferredSharedMemoryCarveout, pc);
      cudaFuncSetAttribute(k_rows3<1, E, kFastRowWarps, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, pc);
      cudaFuncSetAttribute(k_rows3<1, E, kFastRowWarps, 0, kDttCT, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, pc);
    }
  }
  PD_ATTR((k_cols_cm<1, E, fast_col_warps(E), 0>), dtt3_cols_smem<E>());
  PD_ATTR((k_cols_cm<0, E, fast_col_warps(E), 0>), dtt3_cols_smem<E>());
  PD_ATTR((k_cols_cm<1, E, fast_col_warps(E), 1>), dtt3_cols_smem<E>());
  PD_ATTR((k_cols_cm<0, E, fast_col_warps(E), 1>), dtt3_cols_smem<E>());
  PD_ATTR((k_cols3<1, E, fast_col_warps(E), 0>), dtt3_cols_smem<E>());
  PD_ATTR((k_cols3<0, E, fast_col_warps(E), 0>), dtt3_cols_smem<E>());
  PD_ATTR((k_cols3<1, E, fast_col_warps(E), 2>), dtt3_cols_smem<E>());
  PD_ATTR((k_cols3<0, E, fast_col_warps(E), 2>), dtt3_cols_smem<E>());
  if (E == 32) {
    PD_ATTR((k_rows4<1, kPairsPerRowCta>), dttp_rows_smem());
    PD_ATTR((k_rows4<0, kPairsPerRowCta>), dttp_rows_smem());
    PD_ATTR((k_cols4<1>), dttp_cols_smem());
    PD_ATTR((k_cols4<0>), dttp_cols_smem());
  }
  if constexpr (E >= 8) {
    PD_ATTR((k_cols_tma_inv<1, fast_col_warps(E), kYsSlots, E>), dtt3_cols_smem<E>() + 1024 + kYsRing);
    PD_ATTR((k_cols_tma_inv<0, fast_col_warps(E), kYsSlots, E>), dtt3_cols_smem<E>() + 1024 + kYsRing);
  }
  if constexpr (E == 32) {
    PD_ATTR((k_cols_tma_inv<1, fast_col_warps(32), 2>), dtt3_cols_smem<32>() + 1024 + kYsRing / 2);
    PD_ATTR((k_cols_tma_inv<0, fast_col_warps(32), 2>), dtt3_cols_smem<32>() + 1024 + kYsRing / 2);
    PD_ATTR((k_cols_tma_inv<1, fast_col_warps(32), 3>), dtt3_cols_smem<32>() + 1024 + kYsRing * 3 / 4);
    PD_ATTR((k_cols_tma_inv<0, fast_col_warps(32), 3>), dtt3_cols_smem<32>() + 1024 + kYsRing * 3 / 4);
  }
  PD_ATTR((k_cols3<1, E, 4>), ((size_t)4 * Dtt3<1, E>::BUF * sizeof(double)));
  PD_ATTR((k_cols3<0, E, 4>), ((size_t)4 * Dtt3<1, E>::BUF * sizeof(double)));
  return cudaSuccess;
}
#undef PD_ATTR

template <int NEUMANN, int E>
void fast_line_bc(int axis, const double* in, double* out, const LineParams& L, const FastLaunch& F) {
  constexpr int NW = fast_col_warps(E);
  const int C = NW * (32 / E);
  if (E == 32 && F.dtt_ver >= 4 && F.trig2p) {
    if (axis == 0) {
      const unsigned grid = (unsigned)std::min<int64_t>((L.nlines + kPairsPerRowCta - 1) / kPairsPerRowCta, 148 * 4);
      k_rows4<NEUMANN, kPairsPerRowCta><<<grid, kPairsPerRowCta * 64, dttp_rows_smem(), F.stream>>>(in, out, L, F.trig2p);
    } else {
      const int64_t groups = (int64_t)F.nt * ((F.nx + 7) / 8);
      const unsigned grid = (unsigned)std::min<int64_t>(groups, 148);
      k_cols4<NEUMANN><<<grid, 512, dttp_cols_smem(), F.stream>>>(in, out, L, F.trig2p);
    }
    return;
  }
  if (axis == 0) {
    const int64_t groups = (L.nlines + (32 / E) - 1) / (32 / E);
    const unsigned grid = (unsigned)std::min<int64_t>((groups + kFastRowWarps - 1) / kFastRowWarps, 148 * 2);
    // tune 256: pad the dynamic smem so only one CTA (4 warps) fits per SM (occupancy probe)
    const size_t smem = dtt3_rows_smem<E>() + ((L.tune & 256) ? 100 * 1024 : 0);
    const bool gen = L.sin.n || L.sout.n;
    if (gen) k_rows3<NEUMANN, E, kFastRowWarps, 2><<<grid, kFastRowWarps * 32, smem, F.stream>>>(in, out, L, F.trig2);
    else if (L.upd) k_rows3<NEUMANN, E, kFastRowWarps, 3><<<grid, kFastRowWarps * 32, smem, F.stream>>>(in, out, L, F.trig2);
    else if (E == 32 && (L.tune & (1 << 24)) && !L.amax)   // (A/B) the trig tables read every step
      k_rows3<NEUMANN, E, kFastRowWarps, 0, 0><<<grid, kFastRowWarps * 32, smem, F.stream>>>(in, out, L, F.trig2);
    else if (L.amax) k_rows3<NEUMANN, E, kFastRowWarps, 1><<<grid, kFastRowWarps * 32, smem, F.stream>>>(in, out, L, F.trig2);
    else if (NEUMANN && E == 32 && !(L.tune & (1 << 25)) && L.ldi > L.nx && L.ldi % 2 == 0 && ((uintptr_t)in & 15) == 0) {
      if constexpr (NEUMANN && E == 32)      // rows of wp in by bulk copy (x⁻¹); (A/B) tune 2^25: per-element copies
        k_rows3<1, E, kFastRowWarps, 0, kDttCT, 1><<<grid, kFastRowWarps * 32, dtt3_rows_bulk_smem<E>(), F.stream>>>(in, out, L, F.trig2);
    } else k_rows3<NEUMANN, E, kFastRowWarps, 0><<<grid, kFastRowWarps * 32, smem, F.stream>>>(in, out, L, F.trig2);
  } else if (L.tune & 64) {     // 4-warp column CTAs, two per SM (A/B)
    constexpr int C4 = 4 * (32 / E);
    const int64_t groups = (int64_t)F.nt * ((F.nx + C4 - 1) / C4);
    const unsigned grid = (unsigned)std::min<int64_t>(groups, 148 * 2);
    k_cols3<NEUMANN, E, 4><<<grid, 128, (size_t)4 * Dtt3<1, E>::BUF * sizeof(double), F.stream>>>(in, out, L, F.trig2);
  } else {
    const int64_t groups = (int64_t)F.nt * ((F.nx + C - 1) / C);
    const unsigned grid = (unsigned)std::min<int64_t>(groups, 148);
    if (L.sin.n || L.sout.n || L.amax)
      k_cols3<NEUMANN, E, NW, 2><<<grid, NW * 32, dtt3_cols_smem<E>(), F.stream>>>(in, out, L, F.trig2);
    else
      k_cols3<NEUMANN, E, NW, 0><<<grid, NW * 32, dtt3_cols_smem<E>(), F.stream>>>(in, out, L, F.trig2);
  }
}

template <int E>
void fast_line(int neumann, int axis, const double* in, double* out, const LineParams& L, const FastLaunch& F) {
  if (neumann) fast_line_bc<1, E>(axis, in, out, L, F);
  else fast_line_bc<0, E>(axis, in, out, L, F);
}

template <int E>
void fast_time(const double* in, double* out, const TimeParams& T, const FastLaunch& F) {
  if ((T.tune & 128) && fast_time_smem(E, 8) <= 227 * 1024) {   // 8-warp CTAs, one per SM (A/B)
    constexpr int S8 = 2 * (32 / E) * 8;
    const int64_t tiles8 = (F.ns + S8 - 1) / S8;
    const unsigned grid8 = (unsigned)std::min<int64_t>(tiles8, 148);
    k_time2d_v2<E, 8><<<grid8, 256, fast_time_smem(E, 8), F.stream>>>(in, out, T);
    return;
  }
  constexpr int S = 2 * (32 / E) * kFastTimeWarps;
  const int64_t tiles = (F.ns + S - 1) / S;
  const int flags = ((!T.el && !T.l3) ? 1 : 0) | (T.gamma_folded ? 2 : 0);
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, 148 * 8);
  const size_t sm = fast_time_smem(E);
  constexpr int NWT = kFastTimeWarps;
  switch (flags) {
    case 3: k_time2d_v2<E, NWT, 3><<<grid, NWT * 32, sm, F.stream>>>(in, out, T); break;
    case 2: k_time2d_v2<E, NWT, 2><<<grid, NWT * 32, sm, F.stream>>>(in, out, T); break;
    case 1: k_time2d_v2<E, NWT, 1><<<grid, NWT * 32, sm, F.stream>>>(in, out, T); break;
    default: k_time2d_v2<E, NWT, 0><<<grid, NWT * 32, sm, F.stream>>>(in, out, T); break;
  }
}

template <int E>
bool fast_time_tma(double* buf, const TimeParams& T, const FastLaunch& F, const CUtensorMap* tmap) {
  if constexpr (E > 16) {
    return false;
  } else if constexpr (fast_time4_smem<E>() <= 227 * 1024) {      // 3-stage, two groups (k_time2d_v4)
    constexpr int S = 2 * (32 / E) * 4;
    const int64_t tiles = (F.ns + S - 1) / S;
    const unsigned grid = (unsigned)std::min<int64_t>((tiles + 1) / 2, 148);     // tile pairs per CTA
    const int flags = ((!T.el && !T.l3) ? 1 : 0) | (T.gamma_folded ? 2 : 0);
    constexpr size_t sm = fast_time4_smem<E>();
    switch (flags) {
      case 3: k_time2d_v4<E, 3><<<grid, 256, sm, F.stream>>>(*tmap, T); break;
      case 2: k_time2d_v4<E, 2><<<grid, 256, sm, F.stream>>>(*tmap, T); break;
      case 1: k_time2d_v4<E, 1><<<grid, 256, sm, F.stream>>>(*tmap, T); break;
      default: k_time2d_v4<E, 0><<<grid, 256, sm, F.stream>>>(*tmap, T); break;
    }
    return true;
  } else {
    return false;
  }
}

template <int E>
void fast_cols_cm(int neumann, int dir, const double* in, double* out, const LineParams& L, const FastLaunch& F,
                  int64_t lp) {
  constexpr int NW = fast_col_warps(E);
  constexpr int C = NW * (32 / E);
  const int64_t groups = (int64_t)F.nt * ((F.nx + C - 1) / C);
  const unsigned grid = (unsigned)std::min<int64_t>(groups, 148);
  const size_t sm = dtt3_cols_smem<E>();
  if (neumann) {
    if (dir == 0) k_cols_cm<1, E, NW, 0><<<grid, NW * 32, sm, F.stream>>>(in, out, L, F.trig2, lp);
    else k_cols_cm<1, E, NW, 1><<<grid, NW * 32, sm, F.stream>>>(in, out, L, F.trig2, lp);
  } else {
    if (dir == 0) k_cols_cm<0, E, NW, 0><<<grid, NW * 32, sm, F.stream>>>(in, out, L, F.trig2, lp);
    else k_cols_cm<0, E, NW, 1><<<grid, NW * 32, sm, F.stream>>>(in, out, L, F.trig2, lp);
  }
}

template <int E>
bool fast_cols_tma_inv(int neumann, const double* in, const LineParams& L, const FastLaunch& F, int64_t lp,
                       const CUtensorMap* tmo) {
  if constexpr (E < 8) {
    return false;
  } else {
    constexpr int NW = fast_col_warps(E);
    constexpr int C = NW * (32 / E);
    const int64_t groups = (int64_t)F.nt * ((F.nx + C - 1) / C);
    const unsigned grid = (unsigned)std::min<int64_t>(groups, 148);
    // ring slots: 4 (default), 2 or 3 (A/B, M = 2048: tune 2^21 / 2^22; a smaller ring leaves more
    // L1 to the transform's tables — measured slower, 11.4 / 10.9 vs 10.5 ms)
    const int ns = E != 32 ? kYsSlots : (L.tune & (1 << 21)) ? 2 : (L.tune & (1 << 22)) ? 3 : kYsSlots;
    const size_t sm = dtt3_cols_smem<E>() + 1024 + kYsRing / kYsSlots * ns;
#define PD_TI(NS)                                                                                \
    if (neumann) k_cols_tma_inv<1, NW, NS, E><<<grid, NW * 32, sm, F.stream>>>(in, L, F.trig2, lp, *tmo); \
    else k_cols_tma_inv<0, NW, NS, E><<<grid, NW * 32, sm, F.stream>>>(in, L, F.trig2, lp, *tmo);
    if constexpr (E == 32) {
if (ns == 2) { PD_TI(2) } else if (ns == 3) { PD_TI(3) } else { PD_TI(kYsSlots) }
    } else {
      PD_TI(kYsSlots)
    }
#undef PD_TI
    return true;
  }
}

#define PD_FAST_INSTANTIATE(E)                                                                       \
  template void fast_cols_cm<E>(int, int, const double*, double*, const LineParams&, const FastLaunch&, int64_t); \
  template bool fast_time_tma<E>(double*, const TimeParams&, const FastLaunch&, const CUtensorMap*); \
  template bool fast_cols_tma_inv<E>(int, const double*, const LineParams&, const FastLaunch&, int64_t, const CUtensorMap*); \
  template cudaError_t fast_attrs<E>();                                                             \
  template void fast_line<E>(int, int, const double*, double*, const LineParams&, const FastLaunch&); \
  template void fast_time<E>(const double*, double*, const TimeParams&, const FastLaunch&);
#endif

}  // namespace pd
