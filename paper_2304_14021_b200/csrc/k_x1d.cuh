// k_x1d.cuh — 1D long windows with short rows (N_x ≤ 64; c6 has N_x = 63 at N_t = 2^20): the
// x-direction DST-I / DCT-I of every time row as a dense product with the unnormalised eigenbasis
// matrix T (T·T = 2m·I, the oracle's spatial.transform_matrix) on the FP64 tensor cores
// (DMMA m8n8k4), fused with its neighbours in the iteration so the row data crosses HBM once:
//   MODE 0  residual (nested stencils R#15) of U, then r̂ = T r      (U → r̂)
//   MODE 1  r̂ = T r                                                           (apply_precond)
//   MODE 2  δ = T δ̂, ‖δ‖∞                                                      (apply_precond)
//   MODE 3  δ = T δ̂, U += δ, ‖δ‖∞ and ‖U‖∞                                     (iteration)
// The 1/(2m) of T⁻¹ = T/(2m) rides in the time pass's Γ_α⁻¹ scale (k_tlong.cuh).
//
// Both transforms satisfy T[k][n-1-j] = (-1)^k T[k][j] (DST-I and DCT-I alike), so the product
// splits into an even half (k = 2i, from s_j = r_j + r_{n-1-j}) and an odd half (k = 2i+1, from
// d_j = r_j - r_{n-1-j}), each 32 × 32: half the tensor work of the dense 64 × 64 product.
//
// Work unit: 8 consecutive time rows per warp (one m8 tile), warps fully independent (no block
// barriers after the T tiles are staged).  Each warp double-buffers its rows with cp.async: the
// next unit's rows are in flight while the current one is transformed.  Lane j owns the mirrored
// columns j and n-1-j, so s/d (and in MODE 0 the stencil, on ghost-padded rows) need no branches.
// r̂ / δ̂ live in the engine's workspace with an even row pitch (2⌈N_x/2⌉ doubles, pad column 0), so
// the time pass reads and writes them as 16-byte pencil pairs.
#pragma once
#include "common.cuh"
#include "k_residual.cuh"

namespace pd {

constexpr int kX1Warps = 8;               // warps per CTA (2 CTAs per SM)
constexpr int kX1Threads = kX1Warps * 32;
constexpr int kX1H = 32;                  // half transform size (N_x ≤ 64, or 65 Neumann nodes)
constexpr int kX1K = 36;                  // B rows (K): j < 32, plus the centre j = 32 of N_x = 65
constexpr int kX1BP = 40;                 // B tile pitch (doubles): modes i < 32, plus i = 32 (mode 64)
constexpr int kX1RP = 76;                 // staged row pitch: 2 ghosts | up to 65 | 2 ghosts; 76 ≡ 12 (mod 16
                                          // doubles): the 8 rows × 4 columns of a fragment read hit 16 banks twice each
constexpr int kX1In = 9 * kX1RP;          // one input buffer: 9 rows (MODE 0: rows n0-1 .. n0+7)
constexpr size_t kX1Smem = (size_t)(2 * kX1K * kX1BP + kX1Warps * 2 * kX1In) * sizeof(double);

struct X1Params {
  int nx, nt;
  int ld_in, ld_out;         // row pitches (doubles) of in / out
  // time-slab mode (multi-rank long windows): the workspace side (MODE 0/1 out,
  // MODE 2/3 in) in column blocks — column x of row n at (x / bc)·bstride + n·bc + x % bc; bc = 0:
  // the plain pitch layout
  int bc;
  int64_t bstride;
  ResidualParams R;          // stencil coefficients (MODE 0)
  const double* B;           // [2][kX1K][kX1BP]: B[0][j][i] = T[2i][j], B[1][j][i] = T[2i+1][j], zero padded
  DevStats* st;
};

PD_DEV void dmma_f64(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// A u at column x of a ghost-padded row (u = row[x], ghosts at x = -2, -1, n, n+1): nested form
// ((L_{x-1} + L_{x+1}) - 2 L_x) m² with L_y = ((u_{y-1} + u_{y+1}) - 2 u_y) m², the operation order
// of k_residual_1d.  Neumann ghosts are even reflections (L_{-1} = L_1 follows), hinged ghosts the
// odd extension about the boundary node (u_{-1} = 0, u_{-2} = -u_0 ⇒ L_{-1} = 0 exactly).
PD_DEV double x1_applyA(const double* row, int x, const ResidualParams& P) {
  const double um2 = row[x - 2], um1 = row[x - 1], u = row[x], up1 = row[x + 1], up2 = row[x + 2];
  const double Lm = ((um2 + u) - 2.0 * um1) * P.inv_h2;
  const double L0 = ((um1 + up1) - 2.0 * u) * P.inv_h2;
  const double Lp = ((u + up2) - 2.0 * up1) * P.inv_h2;
  const double llap = ((Lm + Lp) - 2.0 * L0) * P.inv_h2;
  return P.kind == 0 ? llap : P.b2 * L0 + P.e2 * llap;
}

template <int MODE>
__global__ void __launch_bounds__(kX1Threads, 2)
k_x1d(const double* __restrict__ u0, const double* __restrict__ in, double* __restrict__ out, X1Params Q) {
  extern __shared__ double xs[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* Bs = xs;                                                  // [2][kX1K][kX1BP]
  double* const ibuf = xs + 2 * kX1K * kX1BP + warp * 2 * kX1In;   // two buffers of kX1In
  for (int i = tid; i < 2 * kX1K * kX1BP; i += kX1Threads) Bs[i] = __ldg(Q.B + i);
  __syncthreads();
  const int nx = Q.nx, nh = nx >> 1;
  // N_x = 65 (Neumann m = 64, c6n): the centre column j = 32 is a ninth K step of the even product
  // and mode 64 a fifth N tile (DCT-I: T[2i][32] = 2(-1)^i, T[64][j] = c_j (-1)^j)
  const bool ext = nx > 2 * kX1H;
  const int nunits = (Q.nt + 7) >> 3;
  // block offsets of this lane's two columns (time-slab input layout)
  const int64_t boff0 = Q.bc ? (int64_t)(lane / Q.bc) * Q.bstride + lane % Q.bc : 0;
  const int64_t boff1 = Q.bc ? (int64_t)((lane + 32) / Q.bc) * Q.bstride + (lane + 32) % Q.bc : 0;
  const int64_t boff2 = Q.bc ? (int64_t)((lane + 64) / Q.bc) * Q.bstride + (lane + 64) % Q.bc : 0;   // N_x = 65
  const int gw = blockIdx.x * kX1Warps + warp, nw = gridDim.x * kX1Warps;
  constexpr int NR = MODE == 0 ? 9 : 8;                             // staged rows per unit
  // cp.async copies of unit `u` (its rows; MODE 0 also row n0-1, = u0 for the first unit) into `b`
  auto fetch = [&](int u, int b) {
    const int n0 = u * 8;
    const int rows = min(8, Q.nt - n0);
    for (int i = 0; i < NR; ++i) {
      const int n = MODE == 0 ? n0 - 1 + i : n0 + i;
      if (n >= n0 + rows) break;
      double* dst = ibuf + b * kX1In + i * kX1RP + 2;
      if (MODE >= 2 && Q.bc) {
        const double* src = in + (size_t)n * Q.bc;
        if (lane < nx) cp_async8(dst + lane, src + boff0);
        if (lane + 32 < nx) cp_async8(dst + lane + 32, src + boff1);
        if (lane + 64 < nx) cp_async8(dst + lane + 64, src + boff2);
      } else {
        const double* src = (MODE == 0 && n < 0) ? u0 : in + (size_t)n * Q.ld_in;
        for (int x = lane; x < nx; x += 32) cp_async8(dst + x, src + x);
      }
    }
  };
  const int g = lane >> 2, q = lane & 3;                            // DMMA fragment coordinates
  double dmax = 0.0;
  unsigned long long ubits = 0ull;
  int cur = 0;
  if (gw < nunits) fetch(gw, 0);
  cp_async_commit();
  for (int u = gw; u < nunits; u += nw) {
    if (u + nw < nunits) fetch(u + nw, cur ^ 1);
    cp_async_commit();
    const int n0 = u * 8, rows = min(8, Q.nt - n0);
    // MODE 3: this lane's U values (row g, columns 2c .. 2c+3 of each n-tile), in flight during the math
    double uv[5][4];
    if (MODE == 3) {
#pragma unroll
      for (int t = 0; t < 5; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int x = 2 * (8 * t + 2 * q) + e;
          uv[t][e] = (g < rows && x < nx) ? out[(size_t)(n0 + g) * Q.ld_out + x] : 0.0;
        }
    }
    cp_async_wait_group<1>();
    __syncwarp();
    double* rb = ibuf + cur * kX1In + 2;                                     // rb[i * kX1RP + x], x = -2 .. nx+1
    if (MODE == 0) {
      // ghost columns of the staged rows (lane i < 9 takes row i)
      if (lane < NR && lane <= rows) {
        double* r = rb + lane * kX1RP;
        if (Q.R.neumann) {
          r[-1] = r[1]; r[-2] = r[2]; r[nx] = r[nx - 2]; r[nx + 1] = r[nx - 3];
        } else {
          r[-1] = 0.0; r[-2] = -r[0]; r[nx] = 0.0; r[nx + 1] = -r[nx - 1];
        }
      }
      __syncwarp();
    }
    // A fragments: row g, columns 4kk + q of s | d, s_j = v_j + v_{n-1-j}, d_j = v_j - v_{n-1-j}
    double as[9], ad[9];
#pragma unroll
    for (int kk = 0; kk < 9; ++kk) {
      const int j = 4 * kk + q, jm = nx - 1 - j;
      const bool pair = j < nh, mid = (j == nh) && (nx & 1);
      double a = 0.0, b = 0.0;
      if (g < rows && (pair || mid)) {
        if (MODE == 0) {
          const double* s = rb + (g + 1) * kX1RP;
          const double* sp = rb + g * kX1RP;
          const double th = Q.R.theta;
          const double dta = (s[j] - sp[j]) * Q.R.inv_dt;
          const double Aa = x1_applyA(s, j, Q.R);
          a = th == 1.0 ? -dta - Aa : -dta - (th * Aa + (1.0 - th) * x1_applyA(sp, j, Q.R));
          if (pair) {
            const double dtb = (s[jm] - sp[jm]) * Q.R.inv_dt;
            const double Ab = x1_applyA(s, jm, Q.R);
            b = th == 1.0 ? -dtb - Ab : -dtb - (th * Ab + (1.0 - th) * x1_applyA(sp, jm, Q.R));
          }
        } else {
          a = rb[g * kX1RP + j];
          if (pair) b = rb[g * kX1RP + jm];
        }
      }
      as[kk] = pair ? a + b : a;
      ad[kk] = pair ? a - b : 0.0;
    }
    __syncwarp();                                   // the buffer is refilled two units from now
    // even modes 2i from s (B[0]), odd modes 2i+1 from d (B[1])
    double ae[5][2], ao[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t) ae[t][0] = ae[t][1] = ao[t][0] = ao[t][1] = 0.0;
    ae[4][0] = ae[4][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const double* be = Bs + (4 * kk + q) * kX1BP + g;
      const double* bo = be + kX1K * kX1BP;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        dmma_f64(ae[t], as[kk], be[8 * t]);
        dmma_f64(ao[t], ad[kk], bo[8 * t]);
      }
      if (ext) dmma_f64(ae[4], as[kk], be[32]);
    }
    if (ext) {                                      // the centre column (K step 9) of the even product
      const double* be = Bs + (32 + q) * kX1BP + g;
#pragma unroll
      for (int t = 0; t < 5; ++t) dmma_f64(ae[t], as[8], be[8 * t]);
    }
    // lane (g, q) holds out[g][2c], out[g][2c+1], out[g][2c+2], out[g][2c+3] for c = 8t + 2q:
    // (ae[t][0], ao[t][0], ae[t][1], ao[t][1])
    if (g < rows) {
      double* dst = out + (size_t)(n0 + g) * Q.ld_out;
#pragma unroll
      for (int t = 0; t < 5; ++t) {
        if (t == 4 && !ext) break;
        const int x = 2 * (8 * t + 2 * q);
        const double v[4] = {ae[t][0], t < 4 ? ao[t][0] : 0.0, ae[t][1], t < 4 ? ao[t][1] : 0.0};
        if (MODE <= 1 && Q.bc) {                    // time-slab blocks (bc even: pairs stay in one block)
          double* bo = out + (size_t)(n0 + g) * Q.bc;
          if (x < Q.ld_out)
            *reinterpret_cast<double2*>(bo + (int64_t)(x / Q.bc) * Q.bstride + x % Q.bc) = make_double2(v[0], v[1]);
          if (x + 2 < Q.ld_out)
            *reinterpret_cast<double2*>(bo + (int64_t)((x + 2) / Q.bc) * Q.bstride + (x + 2) % Q.bc) =
                make_double2(v[2], v[3]);
        } else if (MODE <= 1) {                     // workspace: even pitch, all 64 columns (pad = 0)
          if (x < Q.ld_out) *reinterpret_cast<double2*>(dst + x) = make_double2(v[0], v[1]);
          if (x + 2 < Q.ld_out) *reinterpret_cast<double2*>(dst + x + 2) = make_double2(v[2], v[3]);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (x + e < nx) {
              dmax = amax_acc(dmax, v[e]);
              if (MODE == 3) {
                const double un = uv[t][e] + v[e];
                dst[x + e] = un;
                ubits = max(ubits, (unsigned long long)__double_as_longlong(un) & 0x7fffffffffffffffull);
              } else {
                dst[x + e] = v[e];
              }
            }
        }
      }
    }
    cur ^= 1;
  }
  cp_async_wait_all();
  if (MODE >= 2) warp_atomic_max_abs(&Q.st->dmax_bits, dmax);
  if (MODE == 3) {
    ubits = warp_max_u64(ubits);
    if (lane == 0 && ubits) atomicMax(&Q.st->umax_bits, ubits);
  }
}

}  // namespace pd
