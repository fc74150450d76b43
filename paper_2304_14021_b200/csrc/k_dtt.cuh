// k_dtt.cuh — DCT-I (Neumann) / DST-I (hinged) line passes of Step-(2) in 2D,
// third version.  Mathematics as k_spatial.cuh: a length-M real-to-real
// transform via one complex FFT of H = M/2 points (fft4.cuh, register resident, one warp holds
// P = 32/E lines of M = 64E), then
//   DCT-I: X_{2k} = 2 Re Y_k,  X_{2k+1} = X_1 - 2 Σ_{i=1}^{k} Im Y_i,  X_M = 2 (Re Z_0 - Im Z_0)
//   DST-I: X_{2k} = -2 Im Y_k, X_{2k+1} = Re Y_0 + 2 Σ_{i=1}^{k} Re Y_i
// with Y_k = E_k + W_M^k O_k split from Z_k and conj Z_{H-k}.
//
// What changed against k_fast.cuh (ncu r01a: the line kernels were issue-bound, 3.5 warp
// instructions per point, 45% of them integer overhead):
//   * the prefix sums run in a BLOCKED layout — lane b of a line owns k = 32b .. 32b+31, sums them
//     serially in registers and needs a single segmented warp scan of the 32 block totals per line
//     (before: one 5-step shuffle scan per 32 outputs);
//   * the finished line is written back into the warp buffer (padded, bank-conflict free) and
//     stored with coalesced row (or column-tile) stores — no per-chunk CTA barriers;
//   * the next work item is prefetched into L2 while the current one computes, so HBM streams
//     under the FFT arithmetic even at one or two CTAs per SM;
//   * cos/sin(2πk/M) for the split come from a table laid out [j][b] so a warp's loads coalesce.
#pragma once
#include "common.cuh"
#include "fft4.cuh"
#include "k_spatial.cuh"
#include "tma.cuh"

namespace pd {

// L2 prefetch hints (no data returned; never fault the kernel's own accesses)
PD_DEV void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// one bulk prefetch of [p, p + bytes) rounded out to 16 B and clipped to [.., limit)
PD_DEV void bulk_prefetch_l2(const void* p, size_t bytes, const void* limit) {
  size_t a = (size_t)p & ~(size_t)15, e = ((size_t)p + bytes + 15) & ~(size_t)15;
  const size_t lim = (size_t)limit & ~(size_t)15;
  if (e > lim) e = lim;
  if (e > a) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a)) : "memory");
}

__host__ __device__ constexpr int cmax3(int a, int b, int c) { return a > b ? (a > c ? a : c) : (b > c ? b : c); }

// Trig factors (CT > 0, the default kDttCT = 32): the pre-processing pairs (sin, cos)(π(2n, 2n+1)/M)
// and the split factors (cos, sin)(2πk/M) are loaded exactly every CT-th step and rotated in
// registers in between (one complex product per angle and step, ≤ CT − 1 roundings of a unit
// rotation: a few ulp), so a line reads its three tables once instead of 32 times through L1.
// Measured on c5 (r02, PARADIAG_TUNE A/B of the table (CT = 0), CT = 8 and CT = 32 variants):
// x passes 9.26 → 9.08 → 8.91 ms, y 12.49 → 11.58 → 11.54 ms, y⁻¹ 10.29 → 9.33 → 9.30 ms — the
// line passes are L1-bound (ncu r02za: l1tex 88 % in the row pass, 2.35e9 global-load sectors per
// launch for 0.54e9 of line data) and the FP64 pipe has room for the rotations (29-39 %).
constexpr int kDttCT = 32;
template <int NEUMANN, int E, int CT = kDttCT>
struct Dtt3 {
  static constexpr int P = 32 / E, M = 64 * E, H = 32 * E, LDX = M + 2;
  static constexpr int LOG2H = 5 + ilog2_c(E);
  // output staging: stored index q of line p lives at p*LDO + q + q/64 (64-bit accesses of a
  // half-warp land on 16 distinct banks for the blocked writes and the coalesced reads)
  static constexpr int LDO_MIN = M + E + 1;
  static constexpr int LDO = E >= 16 ? LDO_MIN : ((LDO_MIN + 15) / 16) * 16 + E;
  static constexpr int BUF = (cmax3(2 * kWarpScratch + 2, P * LDX, P * LDO) + 1) & ~1;   // doubles per warp
  PD_DEV static int opos(int q) { return q + (q >> 6); }

  // Transform the P lines held in xb (line p at p*LDX, buffer index 0..M, hinged ends zero) and
  // leave the outputs in xb at p*LDO + opos(stored index).  L.trigs / L.trigc: sin / cos pairs;
  // trig2 = (cos, sin)(2πk/M) stored at [j*E + b] for k = 32b + j.
  // g scales every output (the Γ_α / Γ_α⁻¹·normalisation factor of the line's time slice when the
  // y passes carry it for the time pass; 1 otherwise) at no extra arithmetic.
  PD_DEV static void transform(double* xb, const LineParams& L, const double2* __restrict__ trig2, int lane,
                               double g = 1.0) {
    double2 v[32];
    double x1p[P];
    double2 rot = make_double2(1.0, 0.0);
    if (CT) rot = __ldg(L.trig + 64);                                   // (cos, sin)(64π/M): n -> n + 32
#pragma unroll
    for (int p = 0; p < P; ++p) {
      double acc = 0.0;
      const double* x = xb + p * LDX;
      double2 sn, cs;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int n = lane + 32 * e, j0 = 2 * n;
        const double2 a = *reinterpret_cast<const double2*>(x + j0);   // x_{2n}, x_{2n+1}
        const double m0 = x[M - j0], m1 = x[M - j0 - 1];
        if (!CT || e % (CT > 0 ? CT : 1) == 0) {
          sn = __ldg(L.trigs + n);                                      // sin(π(2n, 2n+1)/M)
          if (NEUMANN || CT) cs = __ldg(L.trigc + n);                   // cos(π(2n, 2n+1)/M)
        } else {                                                        // rotate both angles by 64π/M
          const double c0 = fma(cs.x, rot.x, -sn.x * rot.y), s0 = fma(sn.x, rot.x, cs.x * rot.y);
          const double c1 = fma(cs.y, rot.x, -sn.y * rot.y), s1 = fma(sn.y, rot.x, cs.y * rot.y);
          cs = make_double2(c0, c1);
          sn = make_double2(s0, s1);
        }
        v[p * E + e] = make_double2(ymap<NEUMANN>(a.x, m0, sn.x), ymap<NEUMANN>(a.y, m1, sn.y));
        if (NEUMANN) acc = fma(a.x - m0, cs.x, fma(a.y - m1, cs.y, acc));
      }
      x1p[p] = acc;
    }
    if (NEUMANN) {
#pragma unroll
      for (int p = 0; p < P; ++p) x1p[p] = warp_sum(x1p[p]);
    }
    __syncwarp();
    double2* T = reinterpret_cast<double2*>(xb);
    fft4_s1_to_s2<E, -1>(v, T, LOG2H, L.tw, L.twlog, lane);
    const int pl = lane / E, b = lane - pl * E;
    {
#pragma unroll
      for (int k2 = 0; k2 < 32; ++k2) T[tpad(pl * H + b + E * k2)] = v[k2];   // natural order
    }
    __syncwarp();
    // ---- blocked split + serial prefix: lane (pl, b) owns k = 32b + j
    const double g2 = 2.0 * g;
    double run = 0.0;
    double2 Z0 = make_double2(0.0, 0.0);
    double2 t, r2 = make_double2(1.0, 0.0);
    if (CT) r2 = __ldg(L.trig + 2);                                     // (cos, sin)(2π/M): k -> k + 1
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int k = 32 * b + j;
      const double2 Zk = T[tpad(pl * H + k)];
      const double2 Zm = T[tpad(pl * H + ((H - k) & (H - 1)))];
      const double2 Ev = make_double2(0.5 * (Zk.x + Zm.x), 0.5 * (Zk.y - Zm.y));
      const double2 O = make_double2(0.5 * (Zk.y + Zm.y), -0.5 * (Zk.x - Zm.x));
      if (!CT || j % (CT > 0 ? CT : 1) == 0) t = __ldg(trig2 + j * E + b);
      else t = make_double2(fma(t.x, r2.x, -t.y * r2.y), fma(t.y, r2.x, t.x * r2.y));
      const double Yx = Ev.x + t.x * O.x + t.y * O.y;
      const double Yy = Ev.y + t.x * O.y - t.y * O.x;
      double ev, a;
      if (NEUMANN) {
        ev = g2 * Yx;
        a = k == 0 ? 0.0 : Yy;
      } else {
        ev = -g2 * Yy;
        a = k == 0 ? g * Yx : g2 * Yx;
      }
      run += a;
      v[j] = make_double2(ev, run);
    }
    if (NEUMANN) Z0 = T[tpad(pl * H)];
    // segmented exclusive scan of the block totals over the E lanes of each line
    double incl = run;
#pragma unroll
    for (int o = 1; o < E; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, incl, o);
      if (b >= o) incl += t;
    }
    double excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (b == 0) excl = 0.0;
    double x1 = 0.0;
    if (NEUMANN) {
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (p == pl) x1 = x1p[p];
    }
    const double gx1 = g * x1;
    __syncwarp();                      // every lane has read T: overwrite with the outputs
    double* ob = xb + pl * LDO;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int q = 64 * b + 2 * j;
      if (NEUMANN) {
        ob[opos(q)] = v[j].x;                                  // X_{2k}
        ob[opos(q + 1)] = fma(-g2, excl + v[j].y, gx1);        // X_{2k+1} = g(X_1 - 2 S_k)
      } else {
        ob[opos(q)] = excl + v[j].y;                           // X_{2k+1}: stored index 2k
        if (q > 0) ob[opos(q - 1)] = v[j].x;                   // X_{2k}:   stored index 2k-1
      }
    }
    if (NEUMANN && b == E - 1) ob[opos(M)] = g2 * (Z0.x - Z0.y);    // X_M
    __syncwarp();
  }
};

// Store one staged line (opos layout) to contiguous global memory: 64-element chunks, pointer
// increments only; the optional |v| max is a template switch (no work when it is off).
template <bool AMAX>
PD_DEV void store_line(const double* __restrict__ ob, double* __restrict__ d, int nel, int lane, double& lmax) {
  int q0 = 0;
  d += lane;
  ob += lane;
#pragma unroll 4   // (c5 x 8.97 -> 8.78, x⁻¹ 8.70 -> 8.50 ms: the LDS -> STG latencies of four chunks overlap; 8 loses)
  for (; q0 + 64 <= nel; q0 += 64, ob += 65, d += 64) {
    const double v0 = ob[0], v1 = ob[32];
    d[0] = v0;
    d[32] = v1;
    if (AMAX) lmax = amax_acc(amax_acc(lmax, v0), v1);
  }
  for (int r = 0; q0 + lane + r < nel; r += 32) {
    const double v = ob[r];
    d[r] = v;
    if (AMAX) lmax = amax_acc(lmax, v);
  }
}

// store_line into transpose blocks (SegMap rows form): line ln's elements of block q are contiguous
template <bool AMAX>
PD_DEV void store_line_seg(const double* __restrict__ ob, double* __restrict__ buf, const SegMap& S, int64_t ln,
                           int lane, double& lmax) {
  for (int q = 0; q < S.n; ++q) {
    const int e0 = S.e0[q], e1 = e0 + S.cnt[q];
    double* d = buf + S.off[q] + ln * S.cnt[q] - e0;
    for (int e = e0 + lane; e < e1; e += 32) {
      const double v = ob[e + (e >> 6)];               // opos(e)
      d[e] = v;
      if (AMAX) lmax = amax_acc(lmax, v);
    }
  }
}

// Fused defect-correction update for the last pass (linear kinds, ω = 1): U_line += δ_line with
// δ taken from the staged line (never written to HBM), ‖δ‖∞ and ‖U‖∞ (NaN-safe bit max).  The
// whole U line is loaded into registers first (the transform's registers are dead by now), so
// all of its loads are in flight together.
template <int MAXJ>
PD_DEV void update_line(const double* __restrict__ ob, double* __restrict__ U, int nel, int lane, double& dmax,
                        unsigned long long& ubits) {
  double uv[MAXJ];
#pragma unroll
  for (int j = 0; j < MAXJ; ++j) {
    const int q = lane + 32 * j;
    uv[j] = q < nel ? U[q] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < MAXJ; ++j) {
    const int q = lane + 32 * j;
    if (q < nel) {
      const double d = ob[q + (j >> 1)];          // opos(q): (lane + 32j) >> 6 == j >> 1
      const double u = uv[j] + d;
      U[q] = u;
      dmax = amax_acc(dmax, d);
      ubits = max(ubits, (unsigned long long)__double_as_longlong(u) & 0x7fffffffffffffffull);
    }
  }
}

// ---------------------------------------------------------------- rows (contiguous lines)
// Warps are independent: each takes P consecutive lines per step, prefetches its next group into
// L2, stages the lines with cp.async, transforms and stores them coalesced.
// V: 0 plain (no block I/O, no ‖·‖∞, no fused update), 1 with the ‖·‖∞ epilogue, 2 general
// (runtime block maps / fused update / ‖·‖∞), 3 the fused update (tune 16) — the common passes
// compile without the branches
// BK = 1 (plain Neumann variant reading rows of the padded workspace wp: 16-byte aligned, even
// pitch): the warp's lines arrive by one bulk copy each (lane 0 issues, a per-warp mbarrier
// completes) instead of one 8-byte cp.async per element: c5 x⁻¹ 9.01 -> 8.58 ms.  (The store side
// through per-lane 512-byte bulk stores of a 16-byte aligned staging layout measured 8.96 -> 9.02 ms
// on the forward x pass: not kept.)
// The forward x pass reads the residual at the odd pitch N_x, where every other row starts 8 bytes
// past a 16-byte boundary: starting those rows' bulk copies one double earlier and reading the line
// one double in (the mirrored pair becomes the aligned 16-byte read) is bit-identical but measured
// 8.91 -> 9.51 ms with a second transform instance and 9.05 ms with a warp-uniform branch in the
// pre-processing loop: not kept.  Nor was a de-interleaved staging layout for the per-element copies
// (x_{2i} at xb[i], x_{2i+1} behind them, so all four pre-processing reads are unit-stride: 8
// instead of 12 shared-memory wavefronts per step): bit-identical, 8.90 -> 9.59 ms.
// Occupancy: the register file is per SM sub-partition (16 K registers), so a ninth warp needs
// <= 170 registers per thread; ptxas then takes 168 and spills 96-128 B, and the x passes measured
// 12.6 / 12.0 ms with 9 warps per SM against 8.9 / 8.5 ms with 8 warps at 255 registers.
template <int NEUMANN, int E, int NW, int V = 2, int CT = kDttCT, int BK = 0>
__global__ void __launch_bounds__(NW * 32, 2)
k_rows3(const double* in, double* out, LineParams L, const double2* __restrict__ trig2) {
  static_assert(BK == 0 || (NEUMANN == 1 && V == 0), "bulk row loads: plain Neumann variant only");
  constexpr bool GEN = V == 2;
  constexpr bool UPD = V == 3 || GEN;             // V = 3: the fused update only
  using D = Dtt3<NEUMANN, E, CT>;
  extern __shared__ double2 smem2[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* xb = reinterpret_cast<double*>(smem2) + (size_t)warp * D::BUF;
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(smem2) + (size_t)NW * D::BUF) + warp;
  unsigned phase = 0;
  if (BK) {
    if (lane == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
    }
    __syncwarp();
  }
  double lmax = 0.0;
  unsigned long long ubits = 0ull;
  const int64_t ngroups = (L.nlines + D::P - 1) / D::P;
  const int64_t gstride = (int64_t)gridDim.x * NW;
  const int64_t ldi = GEN ? L.nx : L.ldi, ldo = GEN ? L.nx : L.ldo;   // row pitches (block maps: nx)
  const double* in_end = in + L.nlines * ldi;
  if (!NEUMANN) {
    for (int p = lane; p < D::P; p += 32) {
      xb[p * D::LDX] = 0.0;
      xb[p * D::LDX + D::M] = 0.0;
    }
  }
  for (int64_t g = (int64_t)blockIdx.x * NW + warp; g < ngroups; g += gstride) {
    const int64_t L0 = g * D::P;
    const int64_t rem = L.nlines - L0;
    const int nl = rem < D::P ? (int)rem : D::P;
    const double* src = in + L0 * ldi;
    if ((L.tune & 1) && lane == 0 && g + gstride < ngroups)
      bulk_prefetch_l2(in + (g + gstride) * D::P * ldi, (size_t)D::P * L.nx * sizeof(double), in_end);
    // fused update: bring this group's U rows towards L2 now, they are read after the transform
    if (UPD && L.upd && lane == 0)
      bulk_prefetch_l2(L.upd + L0 * L.nx, (size_t)nl * L.nx * sizeof(double), L.upd + L.nlines * L.nx);
    constexpr unsigned kRowBytes = (unsigned)(D::M + 2) * 8;     // x_0..x_M and one pad double of the row
    if (BK) {                                                  // whole rows of wp by bulk copy
      fence_proxy_async();                                     // the buffer's generic accesses come first
      __syncwarp();
      if (lane == 0) {
        mbar_expect_tx(bar, (unsigned)nl * kRowBytes);
        for (int p = 0; p < nl; ++p)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(smem_u32(xb + p * D::LDX)), "l"(src + p * ldi), "r"(kRowBytes), "r"(smem_u32(bar))
                       : "memory");
      }
      mbar_wait(bar, phase);
      phase ^= 1;
    }
#pragma unroll
    for (int p = 0; p < (BK ? 0 : D::P); ++p) {
      if (p < nl) {
        double* x = xb + p * D::LDX + (NEUMANN ? 0 : 1);
        if (GEN && L.sin.n) {                              // transpose blocks
          for (int q = 0; q < L.sin.n; ++q) {
            const int e0 = L.sin.e0[q], e1 = e0 + L.sin.cnt[q];
            const double* s = in + L.sin.off[q] + (L0 + p) * L.sin.cnt[q] - e0;
            for (int e = e0 + lane; e < e1; e += 32) cp_async8(x + e, s + e);
          }
        } else if (!(L.tune & 16384)) {           // (A/B) tune 16384: no loads
          const double* s = src + p * ldi;
          // (16-byte pair copies from the 16-byte aligned wp rows measured slower: x⁻¹ 9.3 -> 10.3 ms)
          for (int e = lane; e < L.nel; e += 32) cp_async8(x + e, s + e);
        }
      }
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
    if (!NEUMANN) {   // hinged ghosts were overwritten by the previous outputs: restore zeros
      for (int p = lane; p < D::P; p += 32) {
        xb[p * D::LDX] = 0.0;
        xb[p * D::LDX + D::M] = 0.0;
      }
      __syncwarp();
    }
    D::transform(xb, L, trig2, lane);
    double* dst = out + L0 * ldo;
#pragma unroll
    for (int p = 0; p < D::P; ++p) {
      if (p < nl) {
        if (UPD && L.upd) update_line<(D::M + 32) / 32>(xb + p * D::LDO, L.upd + (L0 + p) * L.nx, L.nel, lane, lmax, ubits);
        else if (GEN && L.sout.n && L.amax) store_line_seg<true>(xb + p * D::LDO, out, L.sout, L0 + p, lane, lmax);
        else if (GEN && L.sout.n) store_line_seg<false>(xb + p * D::LDO, out, L.sout, L0 + p, lane, lmax);
        else if (V == 1 || (GEN && L.amax)) store_line<true>(xb + p * D::LDO, dst + p * ldo, L.nel, lane, lmax);
        else if (!(L.tune & 32768)) store_line<false>(xb + p * D::LDO, dst + p * ldo, L.nel, lane, lmax);
      }
    }
    __syncwarp();
  }
  if (V == 1 || ((GEN || V == 3) && L.amax)) warp_atomic_max_abs(L.amax, lmax);
  if (UPD && L.upd) {
    ubits = warp_max_u64(ubits);
    if (lane == 0 && ubits) atomicMax(L.umax, ubits);
  }
  if (GEN && L.sout.n) __threadfence_system();   // block stores may target a peer GPU (peer-memory transposes)
}

// ---------------------------------------------------------------- columns (stride nx)
// CTA = NW warps x P lines = C adjacent columns of one slice.  Rows of the tile are loaded C
// doubles wide (cp.async straight into each column's line buffer), the next tile is prefetched
// into L2 during the transforms, outputs are read back from the line buffers row by row.
template <int NEUMANN, int E, int NW, int V = 2>
__global__ void __launch_bounds__(NW * 32, NW <= 4 ? 2 : 1)
k_cols3(const double* in, double* out, LineParams L, const double2* __restrict__ trig2) {
  constexpr bool GEN = V == 2;
  using D = Dtt3<NEUMANN, E>;
  constexpr int kNel = NEUMANN ? D::M + 1 : D::M - 1;   // stored elements per line (= L.nel)
  constexpr int C = NW * D::P;
  constexpr int NTH = NW * 32;
  extern __shared__ double2 smem2[];
  double* base = reinterpret_cast<double*>(smem2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* xb = base + (size_t)warp * D::BUF;
  const int64_t gx = (L.nx + C - 1) / C;
  const int64_t nsl = L.nlines / L.nx;
  const int64_t ngroups = nsl * gx;
  double lmax = 0.0;
  // thread -> fixed column c = tid % C, rows e = tid / C + k·(NTH / C): pointer increments only
  constexpr int RSTEP = NTH / C;
  static_assert(64 % RSTEP == 0, "row step must divide 64");
  constexpr int PER = 64 / RSTEP;
  const int c_t = threadIdx.x % C, e_t = threadIdx.x / C;
  const int w_t = c_t / D::P, p_t = c_t - w_t * D::P;
  if constexpr (V == 0 || V == 2) {
    if (!(L.tune & 8192)) {
      // Software-pipelined over tiles (plain and block-addressed passes): after the transform every thread copies its
      // outputs from the line buffers into registers (the transform's registers are dead), the CTA
      // syncs, the NEXT tile's cp.async loads go into the freed buffers, and the outputs are stored
      // from registers while those loads are in flight — the store phase of tile G overlaps the
      // load phase of tile G+1 (ncu r01g: ≈ 16 % / 10 % of the samples waited on each).
      constexpr int KB = (kNel + 63) / 64;            // 64-row blocks of a line
      auto issue = [&](int64_t G) {
        const int64_t n = G / gx;
        const int x0 = (int)((G - n * gx) * C);
        const int wcols = (L.tune & 16384) ? 0 : min(C, (int)(L.nx - x0));   // (A/B) tune 16384: no loads
        if (GEN && c_t < wcols && L.sin.n) {           // transpose blocks: row y lives in block s(y)
          double* lb = base + (size_t)w_t * D::BUF + p_t * D::LDX + (NEUMANN ? 0 : 1) + e_t;
          auto seg_base = [&](int sg) {
            return in + L.sin.off[sg] + ((int64_t)n * L.sin.cnt[sg] - L.sin.e0[sg]) * L.nx + x0 + c_t;
          };
          int sg = 0, s_end = L.sin.e0[0] + L.sin.cnt[0];
          const double* sb = seg_base(0);
          for (int e0 = e_t; e0 < kNel; e0 += 64, lb += 64) {
#pragma unroll
            for (int j = 0; j < PER; ++j) {
              const int e = e0 + j * RSTEP;
              if (e < kNel) {
                while (e >= s_end) {
                  ++sg;
                  sb = seg_base(sg);
                  s_end = L.sin.e0[sg] + L.sin.cnt[sg];
                }
                cp_async8(lb + j * RSTEP, sb + (int64_t)e * L.nx);
              }
            }
          }
        } else if (c_t < wcols) {
          double* lb = base + (size_t)w_t * D::BUF + p_t * D::LDX + (NEUMANN ? 0 : 1) + e_t;
          const double* s = in + n * L.ps_in + x0 + (int64_t)e_t * L.nx + c_t;
          const int64_t rstride = (int64_t)RSTEP * L.nx;
          for (int e0 = e_t; e0 < kNel; e0 += 64, lb += 64, s += 64 * L.nx) {
#pragma unroll
            for (int j = 0; j < PER; ++j)
              if (e0 + j * RSTEP < kNel) cp_async8(lb + j * RSTEP, s + j * rstride);
          }
        }
        cp_async_commit();
      };
      if (blockIdx.x < ngroups) issue(blockIdx.x);
      for (int64_t G = blockIdx.x; G < ngroups; G += gridDim.x) {
        const int64_t n = G / gx;
        const int x0 = (int)((G - n * gx) * C);
        const int wcols = min(C, (int)(L.nx - x0));
        if (!NEUMANN) {                               // ghosts (overwritten by the previous outputs)
          for (int p = lane; p < D::P; p += 32) {
            xb[p * D::LDX] = 0.0;
            xb[p * D::LDX + D::M] = 0.0;
          }
        }
        cp_async_wait_all();
        __syncthreads();
        D::transform(xb, L, trig2, lane, L.oscale ? __ldg(L.oscale + n) : 1.0);
        __syncthreads();
        double ov[KB * PER];
        const double* ob = base + (size_t)w_t * D::BUF + p_t * D::LDO + e_t;   // opos(e0 + r) = 65·(e0/64) + r
#pragma unroll
        for (int k = 0; k < KB; ++k)
#pragma unroll
          for (int j = 0; j < PER; ++j)
            ov[k * PER + j] = (c_t < wcols && e_t + 64 * k + j * RSTEP < kNel) ? ob[65 * k + j * RSTEP] : 0.0;
        __syncthreads();                              // every output is in registers: buffers free
        if (G + gridDim.x < ngroups) issue(G + gridDim.x);
        if (GEN && c_t < wcols && L.sout.n) {
          auto seg_base = [&](int sg) {
            return out + L.sout.off[sg] + ((int64_t)n * L.sout.cnt[sg] - L.sout.e0[sg]) * L.nx + x0 + c_t;
          };
          int sg = 0, s_end = L.sout.e0[0] + L.sout.cnt[0];
          double* sb = seg_base(0);
#pragma unroll
          for (int k = 0; k < KB; ++k)
#pragma unroll
            for (int j = 0; j < PER; ++j) {
              const int e = e_t + 64 * k + j * RSTEP;
              if (e < kNel) {
                while (e >= s_end) {
                  ++sg;
                  sb = seg_base(sg);
                  s_end = L.sout.e0[sg] + L.sout.cnt[sg];
                }
                sb[(int64_t)e * L.nx] = ov[k * PER + j];
                if (L.amax) lmax = amax_acc(lmax, ov[k * PER + j]);
              }
            }
        } else if (c_t < wcols && !(L.tune & 32768)) {   // (A/B) tune 32768: no stores
          double* d = out + n * L.ps_out + x0 + (int64_t)e_t * L.nx + c_t;
          const int64_t rstride = (int64_t)RSTEP * L.nx;      // running pointer (see k_cols_cm)
#pragma unroll
          for (int k = 0; k < KB; ++k)
#pragma unroll
            for (int j = 0; j < PER; ++j, d += rstride)
              if (e_t + 64 * k + j * RSTEP < kNel) {
                *d = ov[k * PER + j];
                if (GEN && L.amax) lmax = amax_acc(lmax, ov[k * PER + j]);
              }
        }
      }
      cp_async_wait_all();
      if (GEN && L.amax) warp_atomic_max_abs(L.amax, lmax);
      if (GEN && L.sout.n) __threadfence_system();   // block stores may target a peer GPU
      return;
    }
  }
  if (L.stagger_ns > 0 && blockIdx.x >= gridDim.x / 2) __nanosleep(L.stagger_ns);   // see k_time2d_v2
  for (int64_t G = blockIdx.x; G < ngroups; G += gridDim.x) {
    const int64_t n = G / gx;
    const int x0 = (int)((G - n * gx) * C);
    const int wcols = min(C, (int)(L.nx - x0));
    const double* src = in + n * L.ps_in + x0;
    double* dst = out + n * L.ps_out + x0;
    {
      const int64_t Gn = G + gridDim.x;
      if ((L.tune & 2) && Gn < ngroups) {
        const int64_t nn = Gn / gx;
        const int xn = (int)((Gn - nn * gx) * C);
        const int wn = min(C, (int)(L.nx - xn));
        const double* s = in + nn * L.ps_in + xn;
        const double* lim = in + L.nlines * L.nx;
        if (L.tune & 8) {      // one bulk prefetch per row segment, lane 0 of each warp
          if (lane == 0)
            for (int e = warp; e < kNel; e += NW) bulk_prefetch_l2(s + (int64_t)e * L.nx, (size_t)wn * 8, lim);
        } else {
          for (int e = threadIdx.x; e < kNel; e += NTH) {
            prefetch_l2(s + (int64_t)e * L.nx);
            prefetch_l2(s + (int64_t)e * L.nx + wn - 1);
          }
        }
      }
    }
    if (GEN && c_t < wcols && L.sin.n) {                        // transpose blocks: row y lives in block s(y)
      double* lb = base + (size_t)w_t * D::BUF + p_t * D::LDX + (NEUMANN ? 0 : 1) + e_t;
      auto seg_base = [&](int sg) {
        return in + L.sin.off[sg] + ((int64_t)n * L.sin.cnt[sg] - L.sin.e0[sg]) * L.nx + x0 + c_t;
      };
      int sg = 0, s_end = L.sin.e0[0] + L.sin.cnt[0];
      const double* sb = seg_base(0);
      for (int e0 = e_t; e0 < kNel; e0 += 64, lb += 64) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const int e = e0 + j * RSTEP;
          if (e < kNel) {
            while (e >= s_end) {
              ++sg;
              sb = seg_base(sg);
              s_end = L.sin.e0[sg] + L.sin.cnt[sg];
            }
            cp_async8(lb + j * RSTEP, sb + (int64_t)e * L.nx);
          }
        }
      }
    } else if (c_t < wcols) {
      double* lb = base + (size_t)w_t * D::BUF + p_t * D::LDX + (NEUMANN ? 0 : 1) + e_t;
      const double* s = src + (int64_t)e_t * L.nx + c_t;
      const int64_t rstride = (int64_t)RSTEP * L.nx;
      for (int e0 = e_t; e0 < kNel; e0 += 64, lb += 64, s += 64 * L.nx) {
#pragma unroll
        for (int j = 0; j < PER; ++j)
          if (e0 + j * RSTEP < kNel) cp_async8(lb + j * RSTEP, s + j * rstride);
      }
    }
    cp_async_commit();
    if (!NEUMANN) {
      for (int p = lane; p < D::P; p += 32) {
        xb[p * D::LDX] = 0.0;
        xb[p * D::LDX + D::M] = 0.0;
      }
    }
    cp_async_wait_all();
    __syncthreads();
    D::transform(xb, L, trig2, lane, L.oscale ? __ldg(L.oscale + n) : 1.0);
    __syncthreads();
    if (GEN && c_t < wcols && L.sout.n) {
      const double* ob = base + (size_t)w_t * D::BUF + p_t * D::LDO + e_t;
      auto seg_base = [&](int sg) {
        return out + L.sout.off[sg] + ((int64_t)n * L.sout.cnt[sg] - L.sout.e0[sg]) * L.nx + x0 + c_t;
      };
      int sg = 0, s_end = L.sout.e0[0] + L.sout.cnt[0];
      double* sb = seg_base(0);
      for (int e0 = e_t; e0 < kNel; e0 += 64, ob += 65) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const int e = e0 + j * RSTEP;
          if (e < kNel) {
            while (e >= s_end) {
              ++sg;
              sb = seg_base(sg);
              s_end = L.sout.e0[sg] + L.sout.cnt[sg];
            }
            const double v = ob[j * RSTEP];
            sb[(int64_t)e * L.nx] = v;
            if (GEN && L.amax) lmax = amax_acc(lmax, v);
          }
        }
      }
    } else if (c_t < wcols) {
      const double* ob = base + (size_t)w_t * D::BUF + p_t * D::LDO + e_t;   // opos(e0 + r) = 65·(e0/64) + r
      double* d = dst + (int64_t)e_t * L.nx + c_t;
      const int64_t rstride = (int64_t)RSTEP * L.nx;
      if (V == 1 || (GEN && L.amax)) {
        for (int e0 = e_t; e0 < kNel; e0 += 64, ob += 65, d += 64 * L.nx) {
#pragma unroll
          for (int j = 0; j < PER; ++j)
            if (e0 + j * RSTEP < kNel) {
              const double v = ob[j * RSTEP];
              d[j * rstride] = v;
              lmax = amax_acc(lmax, v);
            }
        }
      } else {
        for (int e0 = e_t; e0 < kNel; e0 += 64, ob += 65, d += 64 * L.nx) {
#pragma unroll
          for (int j = 0; j < PER; ++j)
            if (e0 + j * RSTEP < kNel) d[j * rstride] = ob[j * RSTEP];
        }
      }
    }
    __syncthreads();
  }
  if (V == 1 || (GEN && L.amax)) warp_atomic_max_abs(L.amax, lmax);
  if (GEN && L.sout.n) __threadfence_system();   // block stores may target a peer GPU (peer-memory transposes)
}


// ---------------------------------------------------------------- columns <-> column-major workspace
// The y passes next to the TMA time pass (k_time2d_v4) exchange data with the second workspace wt,
// which holds every slice COLUMN-MAJOR: line x (all y) at wt + n·ps + x·lp, line pitch lp = N_y
// rounded up to even (16-byte aligned lines), slice pitch ps = N_x·lp.  The time pass is pointwise
// in space, and on a square grid the mode eigenvalue λ_p + λ_q is symmetric in (p, q), so it runs
// on this layout unchanged (TimeParams.nx = lp decodes the mode; pads are finite, their output is
// never read).  What changes is the y pass's wt side: one whole contiguous line per warp
// (coalesced, like a row pass) instead of a 64-byte-wide column tile — the forward pass stores its
// lines with store_line, the inverse pass loads them with one 8-byte cp.async per lane and
// element.  The natural-layout side keeps k_cols3's column-tile staging.
// Measured and not kept (round 2, after the trig factors left the tables): a forward variant with 13
// line slots (216 KB) that issues columns 0-4 of the next tile into the 5 free slots right after the
// tile barrier, so only 3/8 of a tile's loads stay exposed between two transforms: parity-green,
// 11.5 -> 18.0 ms on c5.  The per-element cp.async.ca loads land through L1, and a CTA that takes the
// 228 KB shared-memory carve-out leaves 28 KB of it: the lines in flight, not the tables, are what
// the earlier prefetch / ring variants of this pass lost with their L1 (bulk and TMA copies bypass
// it, which is why the inverse pass and the time pass can afford their rings).
// DIR 0: in natural [n][y][x] (slice pitch L.ps_in) -> out column-major wt;
// DIR 1: in column-major wt -> out natural [n][y][x] (slice pitch L.ps_out).  L.upd unused.
template <int NEUMANN, int E, int NW, int DIR, int CT = kDttCT>
__global__ void __launch_bounds__(NW * 32, NW <= 4 ? 2 : 1)
k_cols_cm(const double* in, double* out, LineParams L, const double2* __restrict__ trig2, int64_t lp) {
  using D = Dtt3<NEUMANN, E, CT>;
  constexpr int kNel = NEUMANN ? D::M + 1 : D::M - 1;
  constexpr int C = NW * D::P;
  constexpr int NTH = NW * 32;
  constexpr int RSTEP = NTH / C;
  static_assert(64 % RSTEP == 0, "row step must divide 64");
  constexpr int PER = 64 / RSTEP;
  constexpr int KB = (kNel + 63) / 64;
  extern __shared__ double2 smem2[];
  double* base = reinterpret_cast<double*>(smem2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* xb = base + (size_t)warp * D::BUF;
  const int64_t gx = (L.nx + C - 1) / C;
  const int64_t nsl = L.nlines / L.nx;
  const int64_t ngroups = nsl * gx;
  const int c_t = threadIdx.x % C, e_t = threadIdx.x / C;
  const int w_t = c_t / D::P, p_t = c_t - w_t * D::P;
  const int64_t cps = (int64_t)L.nx * lp;                       // column-major slice pitch
  // DIR 1, Neumann: each wt line (lp doubles, pad included, 16-byte aligned) is ONE bulk copy into
  // its line buffer, completion on an mbarrier (no per-element cp.async issue loop)
  constexpr bool BULK = DIR == 1 && NEUMANN;
  __shared__ uint64_t bar;
  unsigned phase = 0;
  if (BULK) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
  }
  auto issue = [&](int64_t G) {
    const int64_t n = G / gx;
    const int x0 = (int)((G - n * gx) * C);
    const int wcols = min(C, (int)(L.nx - x0));
    if (DIR == 0) {                                               // natural columns -> line buffers
      if (c_t < wcols) {
        double* lb = base + (size_t)w_t * D::BUF + p_t * D::LDX + (NEUMANN ? 0 : 1) + e_t;
        const double* s = in + n * L.ps_in + x0 + (int64_t)e_t * L.ldn + c_t;
        const int64_t rstride = (int64_t)RSTEP * L.ldn;
        for (int e0 = e_t; e0 < kNel; e0 += 64, lb += 64, s += 64 * L.ldn) {
#pragma unroll
          for (int j = 0; j < PER; ++j)
            if (e0 + j * RSTEP < kNel) cp_async8(lb + j * RSTEP, s + j * rstride);
        }
      }
    } else if (BULK) {
      if (threadIdx.x == 0) {
        const int nl = min(C, (int)(L.nx - x0));
        fence_proxy_async();                                      // the buffers' generic reads come first
        mbar_expect_tx(&bar, (unsigned)(nl * lp * 8));
        for (int c = 0; c < nl; ++c) {
          const int w = c / D::P, p = c - w * D::P;
          const double* src = in + n * cps + (int64_t)(x0 + c) * lp;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(smem_u32(base + (size_t)w * D::BUF + p * D::LDX)), "l"(src), "r"((unsigned)(lp * 8)),
                         "r"(smem_u32(&bar)) : "memory");
        }
      }
    } else {                                                      // contiguous wt lines, warp by warp
#pragma unroll
      for (int p = 0; p < D::P; ++p) {
        const int x = x0 + warp * D::P + p;
        if (x < L.nx) {
          double* lb = xb + p * D::LDX + (NEUMANN ? 0 : 1);
          const double* s = in + n * cps + (int64_t)x * lp;
          for (int e = lane; e < kNel; e += 32) cp_async8(lb + e, s + e);
        }
      }
    }
    cp_async_commit();
  };
  if (blockIdx.x < ngroups) issue(blockIdx.x);
  for (int64_t G = blockIdx.x; G < ngroups; G += gridDim.x) {
    const int64_t n = G / gx;
    const int x0 = (int)((G - n * gx) * C);
    const int wcols = min(C, (int)(L.nx - x0));
    if (!NEUMANN) {
      for (int p = lane; p < D::P; p += 32) {
        xb[p * D::LDX] = 0.0;
        xb[p * D::LDX + D::M] = 0.0;
      }
    }
    if (BULK) {
      mbar_wait(&bar, phase);
      phase ^= 1;
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    D::transform(xb, L, trig2, lane, L.oscale ? __ldg(L.oscale + n) : 1.0);
    if (DIR == 0) {
      // each warp takes its staged line(s) into registers (the transform's registers are dead), the
      // CTA syncs, the next tile's loads are issued into the freed buffers, then the lines are stored
      // contiguously into wt (coalesced) while those loads are in flight
      constexpr int NJ = (kNel + 31) / 32;
      double ov[D::P][NJ];
#pragma unroll
      for (int p = 0; p < D::P; ++p)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int q = lane + 32 * j;
          ov[p][j] = q < kNel ? xb[p * D::LDO + q + (q >> 6)] : 0.0;      // opos(q)
        }
      __syncthreads();
      if (G + gridDim.x < ngroups) issue(G + gridDim.x);
#pragma unroll
      for (int p = 0; p < D::P; ++p) {
        const int x = x0 + warp * D::P + p;
        if (x < L.nx) {
          double* d = out + n * cps + (int64_t)x * lp + lane;
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (lane + 32 * j < kNel) d[32 * j] = ov[p][j];
        }
      }
    } else {
      __syncthreads();
      double ov[KB * PER];
      const double* ob = base + (size_t)w_t * D::BUF + p_t * D::LDO + e_t;   // opos(e0 + r) = 65·(e0/64) + r
#pragma unroll
      for (int k = 0; k < KB; ++k)
#pragma unroll
        for (int j = 0; j < PER; ++j)
          ov[k * PER + j] = (c_t < wcols && e_t + 64 * k + j * RSTEP < kNel) ? ob[65 * k + j * RSTEP] : 0.0;
      __syncthreads();
      if (G + gridDim.x < ngroups) issue(G + gridDim.x);
      if (c_t < wcols && !(L.tune & (1 << 19))) {      // (A/B) tune 2^19: no natural-side stores
        // running pointer (rows e_t, e_t + RSTEP, ...): one add per store instead of a 64-bit
        // multiply by the runtime row length (ncu r02t: 12% of the stall samples on those IMADs)
        double* d = out + n * L.ps_out + x0 + (int64_t)e_t * L.ldn + c_t;
        const int64_t rstride = (int64_t)RSTEP * L.ldn;
#pragma unroll
        for (int k = 0; k < KB; ++k)
#pragma unroll
          for (int j = 0; j < PER; ++j, d += rstride)
            if (e_t + 64 * k + j * RSTEP < kNel) *d = ov[k * PER + j];
      }
    }
  }
  cp_async_wait_all();
}

// ---------------------------------------------------------------- y⁻¹ with TMA stores (M = 2048)
// The inverse y pass of k_cols_cm (column-major wt lines in, one bulk copy per Neumann line) with
// the natural-side output leaving through TMA instead of one 8-byte store per element and thread:
// measured on c5 (tune 2^19, r02y), the scattered natural-side stores cost 4.4 of the pass's
// 13.5 ms.  The output goes to the library's padded workspace wp (row pitch L.ldn, a multiple of 8
// doubles, so every 8-column box row is a 64-byte aligned segment and the tensor map's strides are
// legal), through a ring of kYsSlots staging chunks of kYsRows rows × 8 columns: each thread
// writes its outputs of a chunk (a warp covers 4 rows × 64 B: conflict-free), the CTA fences the
// writes to the async proxy and syncs, one thread issues the chunk's box store; before the barrier
// of chunk c that thread waits until the store of chunk c + 1 − kYsSlots has read its slot, so one
// barrier per chunk suffices.  Rows ≥ N_y and columns ≥ N_x of the last boxes are clipped by TMA.
constexpr int kYsRows = 256;
constexpr int kYsSlots = 4;
constexpr size_t kYsRing = (size_t)kYsSlots * kYsRows * 8 * sizeof(double);   // 64 KB

// E = 32 / 16 / 8 (M = 2048 / 1024 / 512): tiles of C = 8 / 16 / 32 columns, staging chunks of
// RC = 256 / 128 / 64 rows (16 KB each), boxes {C, RC, 1}.
template <int E>
__host__ __device__ constexpr int ys_rows() { return kYsRows * 8 / (8 * 32 / E); }

template <int NEUMANN, int NW, int NS = kYsSlots, int E = 32, int CT = kDttCT>
__global__ void __launch_bounds__(NW * 32, 1)
k_cols_tma_inv(const double* in, LineParams L, const double2* __restrict__ trig2, int64_t lp,
               const __grid_constant__ CUtensorMap tmo) {
  using D = Dtt3<NEUMANN, E, CT>;
  constexpr int kNel = NEUMANN ? D::M + 1 : D::M - 1;
  constexpr int C = NW * D::P;
  static_assert(C * 8 <= 256, "box rows of at most 32 doubles");
  constexpr int RC = ys_rows<E>();                              // rows per staging chunk
  constexpr int NTH = NW * 32;
  constexpr int RSTEP = NTH / C;
  constexpr int PER = 64 / RSTEP;
  constexpr int KB = (kNel + 63) / 64;
  constexpr int NCH = (kNel + RC - 1) / RC;
  static_assert(RC % 64 == 0, "a chunk holds whole 64-row blocks");
  constexpr int KPC = RC / 64;                                  // 64-row blocks per chunk
  extern __shared__ double2 smem2[];
  double* base = reinterpret_cast<double*>(smem2);
  double* ring = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(base + (size_t)NW * D::BUF) + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* xb = base + (size_t)warp * D::BUF;
  const int64_t gx = (L.nx + C - 1) / C;
  const int64_t nsl = L.nlines / L.nx;
  const int64_t ngroups = nsl * gx;
  const int c_t = threadIdx.x % C, e_t = threadIdx.x / C;
  const int w_t = c_t / D::P, p_t = c_t - w_t * D::P;
  const int64_t cps = (int64_t)L.nx * lp;
  constexpr bool BULK = NEUMANN;
  __shared__ uint64_t bar;
  unsigned phase = 0;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmo);
    if (BULK) {
      mbar_init(&bar, 1);
      fence_mbar_init();
    }
  }
  __syncthreads();
  auto issue = [&](int64_t G) {
    const int64_t n = G / gx;
    const int x0 = (int)((G - n * gx) * C);
    if (BULK) {
      if (threadIdx.x == 0) {
        const int nl = min(C, (int)(L.nx - x0));
        fence_proxy_async();
        mbar_expect_tx(&bar, (unsigned)(nl * lp * 8));
        for (int c = 0; c < nl; ++c) {
          const int w = c / D::P, p = c - w * D::P;
          const double* src = in + n * cps + (int64_t)(x0 + c) * lp;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(smem_u32(base + (size_t)w * D::BUF + p * D::LDX)), "l"(src), "r"((unsigned)(lp * 8)),
                         "r"(smem_u32(&bar)) : "memory");
        }
      }
    } else {
#pragma unroll
      for (int p = 0; p < D::P; ++p) {
        const int x = x0 + warp * D::P + p;
        if (x < L.nx) {
          double* lb = xb + p * D::LDX + 1;
          const double* s = in + n * cps + (int64_t)x * lp;
          for (int e = lane; e < kNel; e += 32) cp_async8(lb + e, s + e);
        }
      }
    }
    cp_async_commit();
  };
  int64_t chunk = 0;                                            // box stores issued by this CTA
  if (blockIdx.x < ngroups) issue(blockIdx.x);
  for (int64_t G = blockIdx.x; G < ngroups; G += gridDim.x) {
    const int64_t n = G / gx;
    const int x0 = (int)((G - n * gx) * C);
    const int wcols = min(C, (int)(L.nx - x0));
    if (!NEUMANN) {
      for (int p = lane; p < D::P; p += 32) {
        xb[p * D::LDX] = 0.0;
        xb[p * D::LDX + D::M] = 0.0;
      }
    }
    if (BULK) {
      mbar_wait(&bar, phase);
      phase ^= 1;
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    D::transform(xb, L, trig2, lane, L.oscale ? __ldg(L.oscale + n) : 1.0);
    __syncthreads();
    double ov[KB * PER];
    const double* ob = base + (size_t)w_t * D::BUF + p_t * D::LDO + e_t;   // opos(e0 + r) = 65·(e0/64) + r
#pragma unroll
    for (int k = 0; k < KB; ++k)
#pragma unroll
      for (int j = 0; j < PER; ++j)
        ov[k * PER + j] = (c_t < wcols && e_t + 64 * k + j * RSTEP < kNel) ? ob[65 * k + j * RSTEP] : 0.0;
    __syncthreads();                                            // line buffers free: next tile's loads
    if (G + gridDim.x < ngroups) issue(G + gridDim.x);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch, ++chunk) {
      double* slot = ring + (size_t)(chunk % NS) * (RC * C);
#pragma unroll
      for (int kk = 0; kk < KPC; ++kk) {
        const int k = ch * KPC + kk;
        if (k < KB) {
#pragma unroll
          for (int j = 0; j < PER; ++j) slot[(kk * 64 + e_t + j * RSTEP) * C + c_t] = ov[k * PER + j];
        }
      }
      fence_proxy_async();
      if (threadIdx.x == 0) tma_wait_read_le<NS - 2>();         // slot of chunk + 1 free for the next write
      __syncthreads();
      if (threadIdx.x == 0 && !(L.tune & (1 << 19))) {
        tma_store_3d(&tmo, x0, ch * RC, (int)n, slot);
        tma_commit();
      }
    }
  }
  cp_async_wait_all();
  if (threadIdx.x == 0) tma_wait_all();
}

}  // namespace pd
