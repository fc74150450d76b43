// k_fast.cuh — register-resident versions of the 2D hot-path passes (fft4.cuh), for transform
// sizes N = 32·E ≥ 32.  Same mathematics as k_time.cuh / k_spatial.cuh (see there and DESIGN.md
// §5); what changes is the data movement:
//   * a warp holds 1024 complex values in registers (P = 32/E transforms at once);
//   * global tiles are staged with cp.async, each element crosses shared memory once per
//     direction plus one transpose per FFT;
//   * the real-FFT splits / pencil-pair separation read natural-order spectra (conflict-free).
#pragma once
#include "common.cuh"
#include "fft4.cuh"
#include "k_spatial.cuh"
#include "k_time.cuh"
#include "tma.cuh"

namespace pd {

constexpr int kWarpBufD = 2 * kWarpScratch + 2;   // doubles per warp buffer (16-B aligned, bank-skewed)

// Forward time FFT of the warp's PP pencil pairs (stage-1 layout in v), the per-mode divide of
// Step-(2) (Hermitian-paired), and the inverse FFT back to the stage-1 layout.  sw = spatial
// index of the warp's first pencil pair; T = the warp's scratch (kWarpScratch complex).
// tw/twlog, dl: the FFT root table and the d_l table (global, or shared-memory copies).
template <int E, int PP, int FLAGS, bool SMEMTAB = false>
PD_DEV void time_solve_regs(double2 (&v)[32], double2* T, int64_t sw, int lane, const TimeParams& P, double jbar,
                            const double2* tw, int twlog, const double2* dl) {
  constexpr int NT = 32 * E;
  constexpr int LOG2NT = 5 + ilog2_c(E);
  fft4_s1_to_s2<E, -1, SMEMTAB>(v, T, LOG2NT, tw, twlog, lane);
  // ---- per-mode divide (Step-(2)).  lane = (pair pl, k1), v[k2] = Z[l], l = k1 + E k2.  The
  // spectrum is parked in natural order in the warp scratch so every lane reads its Z_{N-l}
  // with the same code path (no divergence, no register hazards).
  const int pl = lane / E, k1 = lane - pl * E;
  const int64_t sa = sw + 2 * pl;
  const double mua = sa < P.ns ? mode_mu(sa, P, jbar) : 0.0;
  const double mub = sa + 1 < P.ns ? mode_mu(sa + 1, P, jbar) : mua;
  const double lama = P.l3 && sa < P.ns ? mode_lam(sa, P) : 0.0;            // PinT-II only
  const double lamb = P.l3 && sa + 1 < P.ns ? mode_lam(sa + 1, P) : lama;
#pragma unroll
  for (int k2 = 0; k2 < 32; ++k2) T[tpad(pl * NT + k1 + E * k2)] = v[k2];
  __syncwarp();
  // Hermitian pairing: d_{N-l} = conj(d_l) and μ is real, so with Af = A_l/(d_l+μa),
  // Bf = B_l/(d_l+μb) the mirror bin is X_{N-l} = conj(Af) + i conj(Bf) — one pair of complex
  // reciprocals serves both bins.  Lane (pl, k1) handles its bins k2 < 16 and their mirrors, which
  // live in the upper half (k2 >= 16) of lane E-k1 (itself for k1 = 0, E/2); the mirrors go
  // through the parked slots.  Bin N/2 (lane k1 = 0, k2 = 16) is its own mirror.
#pragma unroll
  for (int k2 = 0; k2 <= 16; ++k2) {
    if (k2 == 16 && k1 != 0) break;
    const int l = k1 + E * k2;
    const int m = (NT - l) & (NT - 1);
    const double2 Zl = k2 < 16 ? v[k2] : T[tpad(pl * NT + l)];
    const double2 Zm = T[tpad(pl * NT + m)];
    const double2 A = make_double2(0.5 * (Zl.x + Zm.x), 0.5 * (Zl.y - Zm.y));
    const double2 B = make_double2(0.5 * (Zl.y + Zm.y), -0.5 * (Zl.x - Zm.x));
    const double2 d = SMEMTAB ? dl[l] : __ldg(dl + l);
    double2 Af, Bf;
    if (FLAGS & 1) {
      Af = cmul(A, cinv_fast(make_double2(d.x + mua, d.y)));
      Bf = cmul(B, cinv_fast(make_double2(d.x + mub, d.y)));
    } else {
      Af = cmul(A, cinv_fast(shifted(d, P.el, l, mua, P.l3, lama)));
      Bf = cmul(B, cinv_fast(shifted(d, P.el, l, mub, P.l3, lamb)));
    }
    if (k2 < 16) v[k2] = make_double2(Af.x - Bf.y, Af.y + Bf.x);       // X_l = Af + i Bf
    T[tpad(pl * NT + m)] = make_double2(Af.x + Bf.y, Bf.x - Af.y);      // X_{N-l}
  }
  __syncwarp();
#pragma unroll
  for (int k2 = 16; k2 < 32; ++k2) v[k2] = T[tpad(pl * NT + k1 + E * k2)];
  __syncwarp();
  fft4_s2_to_s1<E, +1, SMEMTAB>(v, T, LOG2NT, tw, twlog, lane);
}

// ------------------------------------------------------------------ fused 2D time pass
// CTA = NW warps; warp w owns PP = 32/E pencil pairs = 2·PP spatial points; tile = NT x S.
// FLAGS bit 0 (PLAIN): θ = 1 and no λ₃ term (e_l = 1, the divisor is d_l + μ); bit 1 (FOLD): Γ_α and
// Γ_α⁻¹·normalisation ride on the y passes (P.gamma_folded).  The common c5 case (3) is compiled
// without the optional-table branches and per-element scale loads (time pass 14.15 → 13.6 ms).
template <int E, int NW, int FLAGS = 0>
__global__ void __launch_bounds__(NW * 32, 1)
k_time2d_v2(const double* in, double* out, TimeParams P) {
  constexpr int NT = 32 * E, PP = 32 / E, S = 2 * PP * NW, LD = S + 1;
  constexpr int LOG2NT = 5 + ilog2_c(E);
  extern __shared__ double2 smem2[];
  double* sm = reinterpret_cast<double*>(smem2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* T = smem2 + (size_t)warp * (kWarpBufD / 2);
  const int64_t ntiles = (P.ns + S - 1) / S;
  const double jbar = P.kind >= 2 ? P.st->jbar : 0.0;
  double lmax = 0.0;
  // two CTAs share an SM; starting the second one late puts their load and compute phases out of
  // step, so one streams its tile while the other computes
  if (P.stagger_ns > 0 && blockIdx.x >= gridDim.x / 2) __nanosleep(P.stagger_ns);
  // thread -> fixed point c = tid % S, slices t = tid / S + k·TSTEP: pointer increments only
  // (tiles wider than the CTA, S > 32·NW, only occur for N_t = 32: threads take S/(32·NW) points)
  constexpr int CPT = S > NW * 32 ? S / (NW * 32) : 1;          // points per thread
  constexpr int TSTEP = CPT > 1 ? 1 : NW * 32 / S;
  static_assert(CPT == 1 || S % (NW * 32) == 0, "tile width");
  const int c_t = CPT > 1 ? threadIdx.x : threadIdx.x % S, t_t = CPT > 1 ? 0 : threadIdx.x / S;
  auto issue = [&](int64_t tile) {                  // cp.async of one tile into sm (dead points: 0)
    const int64_t s0 = tile * S;
    if (P.tune & 16384) {                           // (A/B) timing decomposition: no tile loads
      cp_async_commit();
      return;
    }
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc) {
      const int c = c_t + cc * NW * 32;
      const bool live = s0 + c < P.ns;
      double* d = sm + t_t * LD + c;
      const double* g = in + (size_t)t_t * P.ns + s0 + c;
      const size_t gstep = (size_t)TSTEP * P.ns;
#pragma unroll 4
      for (int t = t_t; t < NT; t += TSTEP, d += TSTEP * LD, g += gstep) {
        if (live) cp_async8(d, g);
        else *d = 0.0;
      }
    }
    cp_async_commit();
  };
  // software pipeline over tiles (one point per thread): the outputs go from the tile buffer into
  // registers, the next tile's loads are issued into the freed buffer, then the outputs are stored
  // — the store phase of one tile overlaps the load phase of the next (as k_cols3)
  const bool pipe = CPT == 1 && !(P.tune & 8192);
  if (pipe && blockIdx.x < ntiles) issue(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t s0 = tile * S;
    if (!pipe && (P.tune & 4) && tile + gridDim.x < ntiles) {      // (tune bit 2) L2 prefetch of the CTA's next tile (k_dtt.cuh)
      const int64_t sn = s0 + (int64_t)gridDim.x * S;
      const int64_t last = min((int64_t)S, P.ns - sn) - 1;
      if (P.tune & 8) {
        if (lane == 0)
          for (int t = warp; t < NT; t += NW)
            bulk_prefetch_l2(in + (size_t)t * P.ns + sn, (size_t)(last + 1) * 8, in + (size_t)NT * P.ns);
      } else {
        for (int t = threadIdx.x; t < NT; t += NW * 32) {
          prefetch_l2(in + (size_t)t * P.ns + sn);
          prefetch_l2(in + (size_t)t * P.ns + sn + last);
        }
      }
    }
    if (!pipe) issue(tile);
    cp_async_wait_all();
    __syncthreads();
    double2 v[32];
#pragma unroll
    for (int p = 0; p < PP; ++p) {
      const int c = 2 * (warp * PP + p);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int t = lane + 32 * e;
        const double g = (FLAGS & 2) ? 1.0 : (P.gamma_folded ? 1.0 : __ldg(P.gam + t));
        v[p * E + e] = make_double2(sm[t * LD + c] * g, sm[t * LD + c + 1] * g);
      }
    }
    __syncthreads();
    time_solve_regs<E, PP, FLAGS>(v, T, s0 + 2 * warp * PP, lane, P, jbar, P.tw, P.twlog, P.dl);
    __syncthreads();
#pragma unroll
    for (int p = 0; p < PP; ++p) {
      const int c = 2 * (warp * PP + p);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int t = lane + 32 * e;
        if ((FLAGS & 2) || P.gamma_folded) {
          sm[t * LD + c] = v[p * E + e].x;
          sm[t * LD + c + 1] = v[p * E + e].y;
        } else {
          const double g = __ldg(P.ginv + t);
          sm[t * LD + c] = v[p * E + e].x * g;
          sm[t * LD + c + 1] = v[p * E + e].y * g;
        }
      }
    }
    __syncthreads();
    if (pipe) {
      constexpr int NV = NT / TSTEP;
      double ov[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) ov[k] = sm[(t_t + k * TSTEP) * LD + c_t];
      __syncthreads();                              // the tile buffer is free
      if (tile + gridDim.x < ntiles) issue(tile + gridDim.x);
      if (s0 + c_t < P.ns && !(P.tune & 32768)) {   // (A/B) tune 32768: no tile stores
        double* g = out + (size_t)t_t * P.ns + s0 + c_t;
        const size_t gstep = (size_t)TSTEP * P.ns;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          g[k * gstep] = ov[k];
          if (P.amax) lmax = amax_acc(lmax, ov[k]);
        }
      }
      continue;
    }
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc) {
      const int c = c_t + cc * NW * 32;
      if (s0 + c >= P.ns) continue;
      const double* d = sm + t_t * LD + c;
      double* g = out + (size_t)t_t * P.ns + s0 + c;
      const size_t gstep = (size_t)TSTEP * P.ns;
      if (P.amax) {
#pragma unroll 4
        for (int t = t_t; t < NT; t += TSTEP, d += TSTEP * LD, g += gstep) {
          const double x = *d;
          *g = x;
          lmax = amax_acc(lmax, x);
        }
      } else {
#pragma unroll 4
        for (int t = t_t; t < NT; t += TSTEP, d += TSTEP * LD, g += gstep) *g = *d;
      }
    }
    __syncthreads();
  }
  cp_async_wait_all();
  if (P.amax) warp_atomic_max_abs(P.amax, lmax);
}



// ------------------------------------------------------------------ fused 2D time pass, 3-stage TMA
// Same mathematics and per-group tiling as k_time2d_v2 (a group of 4 warps owns an NT x S tile), but
// one CTA per SM runs TWO groups over THREE tile buffers so the HBM traffic of one tile overlaps the
// FFTs of the others: the CTA's tile k belongs to group k % 2 and buffer k % 3, and after group g has
// stored tile k the buffer receives tile k + 3 (consumed by the other group).  Without loads and
// stores (tune 49152) the c5 time pass takes 8.2 ms against 12.1 ms for k_time2d_v2: the exposed
// memory phases are what this schedule hides.  The tiles move by the Tensor Memory Accelerator
// (with 8-byte cp.async the issue loop took a third of the stall samples and the pass was slower
// than v2, ncu r02f): the pass runs in place on the handle's second
// workspace W2, whose slice pitch ps = N_s rounded up to even makes every tile row 16-byte aligned
// (tma.cuh: an unaligned box start is an illegal instruction).  A tile is NT/RB x S/16 boxes of
// {16 points, RB = min(NT, 256) slices}, SWIZZLE_128B, so the 16-byte pencil-pair reads of 8
// consecutive slices hit 8 distinct bank groups.  One leader thread per group issues the bulk tensor
// stores of its tile and, once they have read shared memory, the loads of the CTA's tile k + 3
// into the same buffer (mbarrier transaction count).  The ragged last tile needs no special case:
// loads past the pitch are zero-filled and stores clipped; the pad column (index N_s) is kept
// finite (zeroed at init) because it shares a complex pencil with point N_s - 1.
template <int E, int FLAGS>
__global__ void __launch_bounds__(256, 1)
k_time2d_v4(const __grid_constant__ CUtensorMap tmap, TimeParams P) {
  constexpr int GW = 4;
  constexpr int NT = 32 * E, PP = 32 / E, S = 2 * PP * GW;
  constexpr int RB = NT < 256 ? NT : 256, NRB = NT / RB, NCH = S / 16;
  constexpr unsigned BOXB = 16u * RB * 8u, TILEB = (unsigned)S * NT * 8u;
  constexpr size_t SCRB = (size_t)GW * kWarpBufD * 8;
  constexpr size_t BUFB = ((TILEB > SCRB ? TILEB : SCRB) + 1023) & ~(size_t)1023;
  static_assert(S % 16 == 0, "TMA time tile");
  extern __shared__ __align__(1024) unsigned char smem_tma[];   // 1024-byte aligned: SWIZZLE_128B boxes
  unsigned char* base = smem_tma;
  double2* s_tw = reinterpret_cast<double2*>(base + 3 * BUFB);
  double2* s_dl = s_tw + NT;
  uint64_t* full = reinterpret_cast<uint64_t*>(s_dl + NT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp / GW, gw = warp - g * GW, gt = threadIdx.x - g * GW * 32;
  const int64_t ntiles = (P.ns + S - 1) / S;
  // tiles 2j, 2j+1 of pair j = blockIdx.x + i·gridDim.x; the CTA's k-th tile is tile_of(k) (< ntiles)
  const int64_t npairs = (ntiles + 1) / 2;
  const int64_t mypairs = npairs > blockIdx.x ? (npairs - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t mine = 2 * mypairs - ((ntiles & 1) && (npairs - 1) % gridDim.x == blockIdx.x ? 1 : 0);
  const double jbar = P.kind >= 2 ? P.st->jbar : 0.0;
  auto gbar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(GW * 32) : "memory"); };
  auto off = [&](int t, int c) -> unsigned {
    return (unsigned)(((c >> 4) * NRB + t / RB) * BOXB) + sw128(t % RB, c & 15);
  };
  // the two groups take neighbouring tiles (2j, 2j+1) of the CTA's pair j: their 128-byte rows share
  // the 256-byte segments the L2 promotes on the first load
  auto tile_of = [&](int64_t k) { return 2 * ((int64_t)blockIdx.x + (k >> 1) * gridDim.x) + (k & 1); };
  auto issue = [&](int64_t k) {                               // one thread: tile k -> buffer k % 3
    unsigned char* buf = base + (size_t)(k % 3) * BUFB;
    mbar_expect_tx(full + k % 3, TILEB);
    const int s0 = (int)(tile_of(k) * S);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
      for (int rb = 0; rb < NRB; ++rb) tma_load_2d(buf + (ch * NRB + rb) * BOXB, &tmap, s0 + 16 * ch, rb * RB, full + k % 3);
  };
  {
    const int sh = P.twlog - (5 + ilog2_c(E));
    for (int i = threadIdx.x; i < NT; i += 256) {
      s_tw[i] = __ldg(P.tw + ((size_t)i << sh));
      s_dl[i] = __ldg(P.dl + i);
    }
  }
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmap);
    for (int b = 0; b < 3; ++b) mbar_init(full + b, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int64_t k = 0; k < 3 && k < mine; ++k) issue(k);
  // the leader waits for its stores to have read the buffer (and issues the next load into it) only
  // after its group has taken the NEXT tile into registers, so the group never waits on the store
  int64_t pend = -1;
  auto flush = [&]() {
    if (gt == 0 && pend >= 0) {
      tma_wait_read_all();
      issue(pend);
    }
    pend = -1;
  };
  for (int64_t k = g; k < mine; k += 2) {
    const int64_t s0 = tile_of(k) * S;
    unsigned char* buf = base + (size_t)(k % 3) * BUFB;
    mbar_wait(full + k % 3, (unsigned)((k / 3) & 1));
    double2 v[32];
#pragma unroll
    for (int p = 0; p < PP; ++p) {
      const int c = 2 * (gw * PP + p);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int t = lane + 32 * e;
        const double2 x = *reinterpret_cast<const double2*>(buf + off(t, c));
        const double gm = (FLAGS & 2) ? 1.0 : (P.gamma_folded ? 1.0 : __ldg(P.gam + t));
        v[p * E + e] = make_double2(x.x * gm, x.y * gm);
      }
    }
    gbar();                                                   // tile in registers: scratch may reuse it
    flush();
    time_solve_regs<E, PP, FLAGS, true>(v, reinterpret_cast<double2*>(buf) + (size_t)gw * (kWarpBufD / 2),
                                        s0 + 2 * gw * PP, lane, P, jbar, s_tw, 5 + ilog2_c(E), s_dl);
    gbar();
#pragma unroll
    for (int p = 0; p < PP; ++p) {
      const int c = 2 * (gw * PP + p);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int t = lane + 32 * e;
        const double gi = ((FLAGS & 2) || P.gamma_folded) ? 1.0 : __ldg(P.ginv + t);
        *reinterpret_cast<double2*>(buf + off(t, c)) = make_double2(v[p * E + e].x * gi, v[p * E + e].y * gi);
      }
    }
    fence_proxy_async();
    gbar();
    if (gt == 0) {
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int rb = 0; rb < NRB; ++rb)
          tma_store_2d(&tmap, (int)s0 + 16 * ch, rb * RB, buf + (ch * NRB + rb) * BOXB);
      tma_commit();
    }
    if (k + 3 < mine) pend = k + 3;                          // buffer k % 3 -> tile k + 3 (see flush)
  }
  flush();
  if (gt == 0) tma_wait_all();
}

}  // namespace pd
