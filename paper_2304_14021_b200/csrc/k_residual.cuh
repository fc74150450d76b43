// k_residual.cuh — all-at-once residual r = b - K(U) (linear) and -G(U) (CH PinT-I,
// P:452-463), nested stencils (R#15), U_0 := u0 folds b in.  Fused reduction: CH Σ(3U² - 1).
#pragma once
#include "common.cuh"

namespace pd {

struct ResidualParams {
  int nx, ny;           // unknowns per axis (ny = 1 in 1D)
  int nt;
  int dim;
  int neumann;          // 1: ghost reflection; 0: hinged zero ghosts (R#14)
  int kind;             // 0 biharmonic, 1 linear CH, 2 CH
  double inv_h2;        // m² exactly
  double inv_dt;        // nt / T
  double b2, e2;        // fl(β·β), fl(ε·ε)
  double theta;         // θ-method: r_n = -(U_n - U_{n-1})/Δt - A(θU_n + (1-θ)U_{n-1}) as
                        // θ·AU_n + (1-θ)·AU_{n-1} (the oracle's order); 1 = backward Euler
  // row slab of a multi-rank run (k_residual_tile only): local rows are global rows
  // [y0g, y0g + ny); rows y0g-2, y0g-1 come from hlo [nt][2][nx], rows y0g+ny, +1 from hhi.
  // Single GPU: y0g = 0, nyg = ny, no halo buffers.
  int y0g, nyg;
  const double* hlo;
  const double* hhi;
  // pipelined solve (k_residual_tile<.., true>): the iterate is U_new = U + dU, formed while staging;
  // U_new is written to unew at the tile's outputs and max |U_new| folded into umax
  const double* dU;
  double* unew;
  unsigned long long* umax;
  // k_residual_tile<.., PADR = true> (opt-in A/B): r is written at row pitch ldr and slice pitch
  // nsr (the padded exchange workspace wp, so the forward x pass can take its rows by bulk copy)
  int64_t ldr, nsr;
};

// Reflect an out-of-range Neumann index back onto the node grid (ghost u_{-1} = u_1).
PD_DEV int reflect(int i, int n) { return i < 0 ? -i : (i >= n ? 2 * (n - 1) - i : i); }

// u at (x, y) of a slice with the BC's ghost rule (x, y may be one layer outside the grid).
PD_DEV double u_at(const double* __restrict__ s, int x, int y, const ResidualParams& P) {
  if (P.neumann) {
    x = reflect(x, P.nx);
    y = P.dim == 2 ? reflect(y, P.ny) : 0;
  } else if (x < 0 || x >= P.nx || (P.dim == 2 && (y < 0 || y >= P.ny))) {
    return 0.0;
  }
  return __ldg(s + (size_t)y * P.nx + x);
}

// Nested discrete Laplacian L(u) at a grid node: ((u_W + u_E) + (u_S + u_N) - 4 u_C) m².
PD_DEV double lap_at(const double* __restrict__ s, int x, int y, const ResidualParams& P) {
  const double c = u_at(s, x, y, P);
  const double we = u_at(s, x - 1, y, P) + u_at(s, x + 1, y, P);
  if (P.dim == 1) return (we - 2.0 * c) * P.inv_h2;
  const double sn = u_at(s, x, y - 1, P) + u_at(s, x, y + 1, P);
  return ((we + sn) - 4.0 * c) * P.inv_h2;
}

// L(u) evaluated at a possibly-ghost position: Neumann reflects (L(u)_{-1} = L(u)_1), hinged
// ghosts of L(u) are 0 (Δu = 0 on the boundary).
PD_DEV bool map_node(int& x, int& y, const ResidualParams& P) {
  if (P.neumann) {
    x = reflect(x, P.nx);
    if (P.dim == 2) y = reflect(y, P.ny);
    return true;
  }
  return !(x < 0 || x >= P.nx || (P.dim == 2 && (y < 0 || y >= P.ny)));
}

PD_DEV double lap_g(const double* __restrict__ s, int x, int y, const ResidualParams& P) {
  return map_node(x, y, P) ? lap_at(s, x, y, P) : 0.0;
}

// CH chemical potential v = u³ - u - ε² L(u) at a possibly-ghost position (Neumann only).
PD_DEV double chem_g(const double* __restrict__ s, int x, int y, const ResidualParams& P) {
  map_node(x, y, P);
  const double u = u_at(s, x, y, P);
  return u * u * u - u - P.e2 * lap_at(s, x, y, P);
}

// One thread per space-time point; grid (ceil(nx/32), ceil(ny/8), nt), block (32, 8).
// r_n = -(U_n - U_{n-1})/Δt - A U_n               (linear, θ = 1)
// r_n = L(U_n³ - U_n - ε² L U_n) - (U_n - U_{n-1})/Δt   (CH)
__global__ void __launch_bounds__(256)
k_residual(const double* __restrict__ u0, const double* __restrict__ U, double* __restrict__ r,
           ResidualParams P, double* __restrict__ jpart) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int n = blockIdx.z;
  const size_t ns = (size_t)P.nx * P.ny;
  const bool live = x < P.nx && y < P.ny;
  double jloc = 0.0;
  if (live) {
    const double* s = U + (size_t)n * ns;
    const double* sp = n == 0 ? u0 : U + (size_t)(n - 1) * ns;
    const size_t idx = (size_t)y * P.nx + x;
    const double uc = __ldg(s + idx);
    const double dtime = (uc - __ldg(sp + idx)) * P.inv_dt;
    double out;
    if (P.kind == 2) {
      double vW = chem_g(s, x - 1, y, P), vE = chem_g(s, x + 1, y, P);
      double vC = chem_g(s, x, y, P);
      double lv;
      if (P.dim == 1) {
        lv = ((vW + vE) - 2.0 * vC) * P.inv_h2;
      } else {
        double vS = chem_g(s, x, y - 1, P), vN = chem_g(s, x, y + 1, P);
        lv = (((vW + vE) + (vS + vN)) - 4.0 * vC) * P.inv_h2;
      }
      out = lv - dtime;
      jloc = 3.0 * uc * uc - 1.0;
    } else {
      auto applyA = [&](const double* q) {
        const double lC = lap_at(q, x, y, P);
        const double lWE = lap_g(q, x - 1, y, P) + lap_g(q, x + 1, y, P);
        double llap;
        if (P.dim == 1) {
          llap = (lWE - 2.0 * lC) * P.inv_h2;
        } else {
          const double lSN = lap_g(q, x, y - 1, P) + lap_g(q, x, y + 1, P);
          llap = ((lWE + lSN) - 4.0 * lC) * P.inv_h2;
        }
        return P.kind == 0 ? llap : P.b2 * lC + P.e2 * llap;
      };
      const double Au = applyA(s);
      out = P.theta == 1.0 ? -dtime - Au : -dtime - (P.theta * Au + (1.0 - P.theta) * applyA(sp));
    }
    r[(size_t)n * ns + idx] = out;
  }
  if (P.kind == 2) {
    // block partial of Σ(3U² - 1) in a fixed order (deterministic): warp sums then warp 0
    __shared__ double wsum[8];
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    double v = warp_sum(jloc);
    if ((tid & 31) == 0) wsum[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int i = 0; i < (int)(blockDim.x * blockDim.y) / 32; ++i) t += wsum[i];
      const size_t bid = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      jpart[bid] = t;
    }
  }
}

// 1D linear residual, one thread per space-time point over the flattened [N_t][N_x] index
// (grid-stride): the same per-point arithmetic as k_residual with a dense thread map, so short
// rows (N_x = 63 at N_t = 2^20, NEXT-3) do not leave most of every block idle.
// Thread map: lanes of a 2^wlog-wide group walk one row (2^wlog ≥ N_x up to 256), 256 >> wlog rows
// per block, grid-stride over rows — no 64-bit division in the index math.
__global__ void __launch_bounds__(256)
k_residual_1d(const double* __restrict__ u0, const double* __restrict__ U, double* __restrict__ r,
              ResidualParams P, int wlog) {
  const int W = 1 << wlog, rpb = 256 >> wlog;
  const int xl = threadIdx.x & (W - 1);
  for (int n = blockIdx.x * rpb + (threadIdx.x >> wlog); n < P.nt; n += gridDim.x * rpb)
  for (int x = xl; x < P.nx; x += W) {
    const size_t i = (size_t)n * P.nx + x;
    const double* s = U + (size_t)n * P.nx;
    const double* sp = n == 0 ? u0 : U + (size_t)(n - 1) * P.nx;
    const double uc = __ldg(s + x);
    const double dtime = (uc - __ldg(sp + x)) * P.inv_dt;
    auto applyA = [&](const double* q) {
      const double lC = lap_at(q, x, 0, P);
      const double llap = ((lap_g(q, x - 1, 0, P) + lap_g(q, x + 1, 0, P)) - 2.0 * lC) * P.inv_h2;
      return P.kind == 0 ? llap : P.b2 * lC + P.e2 * llap;
    };
    const double Au = applyA(s);
    r[i] = P.theta == 1.0 ? -dtime - Au : -dtime - (P.theta * Au + (1.0 - P.theta) * applyA(sp));
  }
}

// J̄ = Σ partials / (N_t N_s), summed by one block in a fixed order.
__global__ void k_jbar_finalize(const double* __restrict__ jpart, size_t np, double inv_count,
                                DevStats* st) {
  __shared__ double sh[1024];
  double t = 0.0;
  for (size_t i = threadIdx.x; i < np; i += blockDim.x) t += jpart[i];
  sh[threadIdx.x] = t;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) st->jbar = sh[0] * inv_count;
}

// ------------------------------------------------------------------------------------------
// 2D row-streaming residual.  A CTA of 128 threads owns one time slice n and a strip of 124
// output columns (+2 halo columns on each side, one column per thread) and streams the
// extended rows -2..ny+1 through a cp.async ring of depth RD: row r is in flight RD rows before
// it is used, so each U element is read from HBM once (halo columns/rows excepted).  The BC
// extension is applied per row/column as a sign: Neumann even reflection (ghost u_{-1} = u_1,
// P:110-117), hinged odd reflection about the boundary node (u = 0 there, Δu = 0 ⇒ L(u) ghosts 0,
// R#14) — evaluating the stencil on the extended grid reproduces the nested definitions exactly.
// L(u) (or v = u³ - u - ε²L(u) for CH) is formed for row r-1, the outer L for row r-2, with the
// x-neighbours exchanged through two double-buffered shared rows.
constexpr int kResStrip = 124;
constexpr int kResRing = 8;

PD_DEV void ext_map(int g, int n, int neumann, int& idx, double& sgn) {
  if (neumann) {
    if (g < 0) g = -g;
    if (g > n - 1) g = 2 * (n - 1) - g;
    idx = min(max(g, 0), n - 1);
    sgn = 1.0;
  } else {
    if (g >= 0 && g < n) { idx = g; sgn = 1.0; }
    else if (g == -1 || g == n) { idx = 0; sgn = 0.0; }
    else if (g < -1) { idx = min(-g - 2, n - 1); sgn = -1.0; }
    else { idx = max(2 * n - g, 0); sgn = -1.0; }
  }
}

__global__ void __launch_bounds__(128)
k_residual_2d(const double* __restrict__ u0, const double* __restrict__ U, double* __restrict__ r,
              ResidualParams P, double* __restrict__ jpart) {
  __shared__ double ring_u[kResRing][128];
  __shared__ double ring_p[kResRing][128];
  __shared__ double su[2][128];
  __shared__ double sv[2][128];
  __shared__ double wsum[4];
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * kResStrip;
  const int n = blockIdx.y;
  const size_t ns = (size_t)P.nx * P.ny;
  const double* s = U + (size_t)n * ns;
  const double* sp = n == 0 ? u0 : U + (size_t)(n - 1) * ns;
  const int gx = x0 - 2 + tid;
  int cx;
  double sxg;
  ext_map(gx, P.nx, P.neumann, cx, sxg);
  const bool outcol = tid >= 2 && tid < kResStrip + 2 && gx < P.nx;
  const int nrows = P.ny + 4;             // extended rows, grid row = r - 2
  const bool ch = P.kind == 2;

  auto issue = [&](int rr) {              // copies for iteration rr: u ext row rr, prev grid row rr-4
    if (rr < nrows) {
      int cy;
      double sy;
      ext_map(rr - 2, P.ny, P.neumann, cy, sy);
      cp_async8(&ring_u[rr % kResRing][tid], s + (size_t)cy * P.nx + cx);
      const int pr = rr - 4;
      if (outcol && pr >= 0 && pr < P.ny) cp_async8(&ring_p[rr % kResRing][tid], sp + (size_t)pr * P.nx + gx);
    }
    cp_async_commit();
  };
#pragma unroll 1
  for (int rr = 0; rr < kResRing; ++rr) issue(rr);

  double u_m2 = 0, u_m1 = 0;              // u at ext rows r-2, r-1
  // at the top of iteration rr: u_m1/u_m2 = u at ext rows rr-1/rr-2; v_m1/v_m2 = inner value at ext
  // rows rr-2/rr-3 (computed one iteration later than u); L_m1 = L(u) at ext row rr-2
  double v_m2 = 0, v_m1 = 0;
  double L_m1 = 0;
  double jloc = 0.0;
  for (int rr = 0; rr < nrows; ++rr) {
    cp_async_wait_group<kResRing - 1>();
    int cy;
    double sy;
    ext_map(rr - 2, P.ny, P.neumann, cy, sy);
    const double uc = ring_u[rr % kResRing][tid] * (sxg * sy);
    const double uprev = ring_p[rr % kResRing][tid];
    issue(rr + kResRing);
    su[rr & 1][tid] = uc;
    __syncthreads();
    // inner stage at ext row rr-1: L(u), or v = u³ - u - ε² L(u) for CH
    double inner = 0.0, Lr = 0.0;
    if (rr >= 2 && tid >= 1 && tid < 127) {
      const double* row = su[(rr - 1) & 1];
      Lr = ((row[tid - 1] + row[tid + 1]) + (u_m2 + uc) - 4.0 * u_m1) * P.inv_h2;
      inner = ch ? u_m1 * u_m1 * u_m1 - u_m1 - P.e2 * Lr : Lr;
    }
    sv[(rr - 1) & 1][tid] = inner;
    __syncthreads();
    // outer stage at ext row rr-2 (grid row rr-4)
    if (rr >= 4 && outcol) {
      const double* row = sv[(rr - 2) & 1];
      const double outer = ((row[tid - 1] + row[tid + 1]) + (v_m2 + inner) - 4.0 * v_m1) * P.inv_h2;
      const double uo = u_m2;               // u at ext row rr-2
      const double dtime = (uo - uprev) * P.inv_dt;
      double out;
      if (ch) {
        out = outer - dtime;
        jloc += 3.0 * uo * uo - 1.0;
      } else {
        const double Au = P.kind == 0 ? outer : P.b2 * L_m1 + P.e2 * outer;
        out = -dtime - Au;
      }
      r[(size_t)n * ns + (size_t)(rr - 4) * P.nx + gx] = out;
    }
    u_m2 = u_m1; u_m1 = uc;
    v_m2 = v_m1; v_m1 = inner;
    L_m1 = Lr;
  }
  cp_async_wait_all();
  if (ch) {
    const double v = warp_sum(jloc);
    if ((tid & 31) == 0) wsum[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) jpart[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = (wsum[0] + wsum[1]) + (wsum[2] + wsum[3]);
  }
}

}  // namespace pd

namespace pd {

// ------------------------------------------------------------------------------------------
// 2D residual, tiled and time-marching (v2).  ncu r01b: the row-streaming kernel above issued 5.5
// warp instructions per point (ring indexing, per-row BC maps, two barriers per row).  Here a CTA
// owns a TY x TX output tile and marches over a chunk of time slices n0..n1-1:
//   * the BC-extended tile of U_n (2-point halo; the even/odd extension signs of ext_map, hence the
//     same nested ghost rules R#14/R#15) is staged with cp.async into one of two buffers while the
//     previous slice computes — the per-element source offsets and signs are computed once;
//   * U_{n-1} at the tile's outputs is kept in registers from the previous slice (only the chunk's
//     first slice reads it from global), so U is read from HBM once;
//   * inner values L(u) (CH: v = u³ - u - ε²L(u)) on the 1-point-haloed tile go to shared memory,
//     then the outer stencil and the time difference.  Arithmetic and evaluation order are those of
//     k_residual_2d.
constexpr int kResTX = 62, kResTY = 32, kResThreads = 256, kResChunk = 32;
constexpr int kResUX = kResTX + 4, kResUY = kResTY + 4;     // staged U tile (66 x 36)
constexpr int kResIX = kResTX + 2, kResIY = kResTY + 2;     // inner-value tile (64 x 34)
constexpr int kResUP = kResUX + 1, kResIP = kResIX + 1;     // pitches (odd: conflict-free columns)
constexpr int kResUN = kResUY * kResUX;                     // staged elements
constexpr int kResPer = (kResUN + kResThreads - 1) / kResThreads;
constexpr int kResGroups = kResThreads / kResIX;            // 4 row groups of the 64 inner columns
constexpr int kResOut = kResTY / kResGroups;                // 8 consecutive output rows per thread
constexpr size_t kResSmem = (2 * (size_t)kResUY * kResUP + (size_t)kResIY * kResIP) * sizeof(double);
constexpr size_t kResSmemUpd = (4 * (size_t)kResUY * kResUP + (size_t)kResIY * kResIP) * sizeof(double);
static_assert(kResIX * kResGroups == kResThreads, "one thread per inner column and row group");

// MODE 0: backward Euler (linear, CH PinT-I); 1: θ-method (A U_{n-1} term, NEXT-2); 2: CH PinT-II
// (Eyre, NEXT-1: inner v = U³ - ε²L(U), r = (L(v) - L(U_{n-1})) - (U_n - U_{n-1})/Δt, Σ 3U²).
// Modes 1 and 2 carry a previous-slice quantity (A U_{n-1} / L U_{n-1}) in registers.
// Threads stream down vertical strips (thread = one column x one row group) so the vertical
// neighbours of both stencils stay in registers: 3 shared loads per inner value, 3-4 per output
// (ncu r01c: the 2D-loop version spent 2.9 warp instructions per point).
// UPD (pipelined solve, linear kinds): the previous iteration's update is applied here — the
// staged tile is U + dU, the outputs also write U_new to P.unew (a different buffer: neighbouring
// tiles still read the old iterate as their halo) and reduce ‖U_new‖∞.
// VAR: 0 general (runtime CH / slab-halo checks), 1 linear kind on a single handle, 3 linear kind on
// a slab (halo rows, no CH branch), 2 CH kind on a
// single handle — the single-handle variants are compiled without those branches
template <int MODE, bool UPD = false, int VAR = 0, bool PADR = false>
__global__ void __launch_bounds__(kResThreads)
k_residual_tile(const double* __restrict__ u0, const double* __restrict__ U, double* __restrict__ r,
                ResidualParams P, double* __restrict__ jpart) {
  extern __shared__ double2 smem2[];
  double* const sU0 = reinterpret_cast<double*>(smem2);
  double* const sU1 = sU0 + kResUY * kResUP;
  double* const sI = sU1 + kResUY * kResUP;
  double* const sD0 = sI + kResIY * kResIP;            // UPD: staged dU tiles
  double* const sD1 = sD0 + kResUY * kResUP;
  unsigned long long ubits = 0ull;
  __shared__ double wsum[kResThreads / 32];
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * kResTX, y0 = blockIdx.y * kResTY;
  const int n0 = blockIdx.z * kResChunk, n1 = min(n0 + kResChunk, P.nt);
  const size_t ns = (size_t)P.nx * P.ny;
  const bool ch = (VAR == 1 || VAR == 3) ? false : (VAR == 2 ? true : P.kind >= 2);
  constexpr bool eyre = MODE == 2;
  const bool halos = (VAR == 1 || VAR == 2) ? false : (P.hlo != nullptr || P.hhi != nullptr);
  // staging map (slice independent): element k of this thread -> smem slot, source buffer
  // (0: U, 1: lower halo, 2: upper halo) and offset within its slice, extension sign
  int soff[kResPer], dpos[kResPer], ssel[kResPer];
  double sgn[kResPer];
#pragma unroll
  for (int k = 0; k < kResPer; ++k) {
    const int i = tid + k * kResThreads;
    const int ry = i / kResUX, rx = i - ry * kResUX;
    int cy = 0, cx = 0, sel = 0;
    double sy = 0.0, sg = 0.0;
    if (i < kResUN) {
      ext_map(P.y0g + y0 - 2 + ry, P.nyg, P.neumann, cy, sy);     // global row
      ext_map(x0 - 2 + rx, P.nx, P.neumann, cx, sg);
      cy -= P.y0g;                                                // local row
      if (sy == 0.0) cy = 0;            // hinged boundary line: zeroed by the sign; load any local row
      if (cy < 0) { sel = 1; cy += 2; }
      else if (cy >= P.ny) { sel = 2; cy -= P.ny; }
    }
    soff[k] = i < kResUN ? cy * P.nx + cx : -1;
    ssel[k] = sel;
    dpos[k] = ry * kResUP + rx;
    sgn[k] = sy * sg;
  }
  const size_t hstride = 2 * (size_t)P.nx;
  auto stage = [&](double* dst, int n) {           // n = -1: u0 (single-GPU warm-up slice)
    const double* b0 = n < 0 ? u0 : U + (size_t)n * ns;
    if (UPD && n >= 0) {                              // the dU tile of the same slice
      double* dd = dst == sU0 ? sD0 : sD1;
      const double* d0 = P.dU + (size_t)n * ns;
#pragma unroll
      for (int k = 0; k < kResPer; ++k)
        if (soff[k] >= 0) cp_async8(dd + dpos[k], d0 + soff[k]);
    }
    if (!halos) {
#pragma unroll
      for (int k = 0; k < kResPer; ++k)
        if (soff[k] >= 0) cp_async8(dst + dpos[k], b0 + soff[k]);
    } else {
#pragma unroll
      for (int k = 0; k < kResPer; ++k)
        if (soff[k] >= 0) {
          const double* b = ssel[k] == 0 ? b0 : (ssel[k] == 1 ? P.hlo : P.hhi) + (size_t)n * hstride;
          cp_async8(dst + dpos[k], b + soff[k]);
        }
    }
    cp_async_commit();
  };
  auto fix_signs = [&](double* dst, int n) {     // U + dU (UPD), then the hinged odd extension
    if (UPD && n >= 0) {
      const double* dd = dst == sU0 ? sD0 : sD1;
#pragma unroll
      for (int k = 0; k < kResPer; ++k)
        if (soff[k] >= 0) dst[dpos[k]] += dd[dpos[k]];
    }
    if (!P.neumann) {
#pragma unroll
      for (int k = 0; k < kResPer; ++k)
        if (soff[k] >= 0) dst[dpos[k]] *= sgn[k];
    }
  };
  // inner strip: inner column ix = tid % 64, rows [ir0, ir1) of the 34 inner rows
  const int ix = tid % kResIX, grp = tid / kResIX;
  const int ir0 = (grp * kResIY) / kResGroups, ir1 = ((grp + 1) * kResIY) / kResGroups;
  // output strip: column tx = ix (< TX), rows ty0 .. ty0+7
  const int tx = ix, ty0 = grp * kResOut;
  const int gx = x0 + tx;
  const bool xout = tx < kResTX && gx < P.nx;
  double prev[kResOut];
  {
    const double* sp = n0 == 0 ? u0 : U + (size_t)(n0 - 1) * ns;
#pragma unroll
    for (int j = 0; j < kResOut; ++j) {
      const int gy = y0 + ty0 + j;
      const size_t o = (size_t)gy * P.nx + gx;
      prev[j] = (xout && gy < P.ny) ? __ldg(sp + o) + (UPD && n0 > 0 ? __ldg(P.dU + (size_t)(n0 - 1) * ns + o) : 0.0)
                                    : 0.0;
    }
  }
  // PADR: this thread's first output of slice 0 (row pitch ldr, slice pitch nsr)
  double* const rpad = r + (size_t)(y0 + ty0) * (size_t)(PADR ? P.ldr : 0) + gx;
  double jloc = 0.0;
  // θ < 1 / PinT-II need A U_{n-1} / L U_{n-1}: march one extra (output-free) slice n0-1 first;
  // the quantity of every slice is then carried to the next in registers like U_{n-1}
  constexpr bool thet = MODE != 0;
  const int nstart = thet ? n0 - 1 : n0;
  double prevA[kResOut];
#pragma unroll
  for (int j = 0; j < kResOut; ++j) prevA[j] = 0.0;
  stage(sU0, nstart);
  for (int n = nstart; n < n1; ++n) {
    double* cur = ((n - nstart) & 1) ? sU1 : sU0;
    double* nxt = ((n - nstart) & 1) ? sU0 : sU1;
    cp_async_wait_all();
    fix_signs(cur, n);
    __syncthreads();                       // cur staged; previous slice done with nxt and sI
    if (n + 1 < n1) stage(nxt, n + 1);
    // ---- inner values down the strip: u rows stream through registers
    {
      const double* c = cur + (ir0 + 1) * kResUP + (ix + 1);
      double ua = c[-kResUP], uc = c[0];
      double* out = sI + ir0 * kResIP + ix;
      for (int iy = ir0; iy < ir1; ++iy, c += kResUP, out += kResIP) {
        const double ub = c[kResUP];
        const double Lr = ((c[-1] + c[1]) + (ua + ub) - 4.0 * uc) * P.inv_h2;
        *out = eyre ? uc * uc * uc - P.e2 * Lr : (ch ? uc * uc * uc - uc - P.e2 * Lr : Lr);
        ua = uc;
        uc = ub;
      }
    }
    __syncthreads();
    // ---- outer stencil + time difference down the output strip
    double* rn = PADR ? rpad + (size_t)max(n, 0) * (size_t)P.nsr : r + (size_t)max(n, 0) * ns;
    if (tx < kResTX) {
      const double* I = sI + (ty0 + 1) * kResIP + (tx + 1);
      const double* cu = cur + (ty0 + 2) * kResUP + (tx + 2);
      double Ia = I[-kResIP], Ic = I[0];
#pragma unroll
      for (int j = 0; j < kResOut; ++j, I += kResIP, cu += kResUP) {
        const double Ib = I[kResIP];
        const int gy = y0 + ty0 + j;
        const double uo = cu[0];
        const double outer = ((I[-1] + I[1]) + (Ia + Ib) - 4.0 * Ic) * P.inv_h2;
        const double dtime = (uo - prev[j]) * P.inv_dt;
        double outv;
        if (eyre) {
          const double Lc = ((cu[-1] + cu[1]) + (cu[-kResUP] + cu[kResUP]) - 4.0 * uo) * P.inv_h2;
          outv = (outer - prevA[j]) - dtime;
          prevA[j] = Lc;
          if (n >= n0 && gx < P.nx && gy < P.ny) jloc += 3.0 * uo * uo;
        } else if (ch) {
          outv = outer - dtime;
          if (n >= n0 && gx < P.nx && gy < P.ny) jloc += 3.0 * uo * uo - 1.0;
        } else {
          const double Au = P.kind == 0 ? outer : P.b2 * Ic + P.e2 * outer;
          outv = thet ? -dtime - (P.theta * Au + (1.0 - P.theta) * prevA[j]) : -dtime - Au;
          if (thet) prevA[j] = Au;
        }
        if (n >= n0 && gx < P.nx && gy < P.ny) {
          if (PADR) rn[(size_t)j * (size_t)P.ldr] = outv;
          else rn[(size_t)gy * P.nx + gx] = outv;
          if (UPD) {
            P.unew[(size_t)n * ns + (size_t)gy * P.nx + gx] = uo;
            ubits = max(ubits, (unsigned long long)__double_as_longlong(uo) & 0x7fffffffffffffffull);
          }
        }
        prev[j] = uo;
        Ia = Ic;
        Ic = Ib;
      }
    }
  }
  if (UPD) {
    ubits = warp_max_u64(ubits);
    if ((tid & 31) == 0 && ubits) atomicMax(P.umax, ubits);
  }
  if (ch) {
    const double v = warp_sum(jloc);
    if ((tid & 31) == 0) wsum[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kResThreads / 32; ++w) t += wsum[w];
      jpart[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
  }
}

}  // namespace pd
