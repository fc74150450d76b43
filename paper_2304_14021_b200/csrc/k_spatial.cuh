// k_spatial.cuh — DCT-I (Neumann) / DST-I (hinged) along one axis of every time slice.
//
// Step-(2) of P:162 in 2D diagonalises Δ_h with the unnormalised real-to-real transforms
// (P:233):
//   DCT-I  X_k = x_0 + (-1)^k x_M + 2 Σ_{j=1}^{M-1} x_j cos(πjk/M),   k = 0..M   (Neumann nodes)
//   DST-I  X_k = 2 Σ_{j=1}^{M-1} x_j sin(πjk/M),                        k = 1..M-1 (hinged interior)
// Both are self-inverse up to 2M, so the same kernels serve the forward and inverse passes (the
// 1/(2M) factors are folded into the time pass).  M = m is a power of two.
//
// Algorithm (one warp per line): a real sequence y of length M is built from x and
// its mirror, y_j = ½(x_j + x_{M-j}) - s_j (x_j - x_{M-j}) (DCT) or s_j (x_j + x_{M-j}) + ½(x_j - x_{M-j})
// (DST), s_j = sin(πj/M), packed in place as M/2 complex z_n = y_{2n} + i y_{2n+1}; the warp FFT
// (DIF, output bit-reversed) gives Z; the real FFT splits as Y_k = E_k + W_M^k O_k and
//   DCT-I: X_{2k} = 2 Re Y_k, X_{2k+1} = X_1 - 2 Σ_{i=1}^{k} Im Y_i, X_1 = Σ_j (x_j - x_{M-j}) cos(πj/M)
//   DST-I: X_{2k} = -2 Im Y_k, X_{2k+1} = Re Y_0 + 2 Σ_{i=1}^{k} Re Y_i
// with the prefix sums done as warp scans over the interleaved k layout.
//
// Rows (x axis, contiguous) use one warp per row; columns (y axis, stride n_x) use a CTA of W warps
// on W adjacent columns, loading W-wide row segments and staging outputs for coalesced stores.
// Lines are staged in shared memory with cp.async (all copies in flight at once).
#pragma once
#include "common.cuh"
#include "fft.cuh"

namespace pd {

// Transpose-block addressing of a line pass's input or output (multi-rank slab mode):
// the all-to-all send / receive buffers hold one block per peer, so the passes next to a transpose
// read or write the blocks directly instead of the slab plus a pack / unpack copy.
//   rows (x pass):    element x ∈ [e0[q], e0[q]+cnt[q]) of local line ln at buf[off[q] + ln·cnt[q] + x - e0[q]]
//   columns (y pass): row y ∈ [e0[s], e0[s]+cnt[s]) of slice n, column c at
//                     buf[off[s] + (n·cnt[s] + y - e0[s])·nxl + c]
// n == 0: plain slab addressing.
constexpr int kMaxSeg = 8;
struct SegMap {
  int n;
  int e0[kMaxSeg];
  int cnt[kMaxSeg];
  int64_t off[kMaxSeg];
};

struct LineParams {
  int64_t nlines;        // rows: nt·ny;  columns: nt·nx
  int64_t nx, ns;        // row length (elements) and slice size
  int nel;               // stored elements per line: M+1 (Neumann) or M-1 (hinged)
  int M, log2h;          // M = m (intervals); H = M/2 complex points
  const double2* trig;   // trig[j] = (cos(πj/M), sin(πj/M)), j = 0..M
  const double2* trigs;  // k_dtt.cuh: trigs[n] = (sin(2nπ/M), sin((2n+1)π/M)), n < M/2 (one
  const double2* trigc;  //   contiguous 16-byte load per lane); trigc[n] likewise with cos
  const double2* tw;     // FFT twiddles exp(-2πik/2^twlog)
  int twlog;
  unsigned long long* amax;   // optional: max |out| (NULL = off)
  int tune;              // PARADIAG_TUNE bits (A/B switches for measurements; 0 = defaults)
  double* upd;           // k_rows3 only: fused update U += out (out not stored), NULL = off
  unsigned long long* umax;   // with upd: max |U| after the update (bit-pattern max, NaN-safe)
  const double* oscale;  // k_cols3 only: outputs of slice n scaled by oscale[n] (NULL = 1)
  int stagger_ns;        // k_cols3: start delay of the second CTA of each SM (phase offset)
  SegMap sin, sout;      // k_rows3 / k_cols3: transpose-block input / output (n = 0: plain)
  int64_t ps_in, ps_out; // k_cols3: slice pitch of in / out (ns, or the even pitch of the TMA workspace)
  int64_t ldi, ldo;      // k_rows3 (plain variants): row pitch of in / out (nx, or the padded pitch of wp)
  int64_t ldn;           // k_cols_cm: row pitch of the natural-layout side (nx, or the padded pitch of wp)
};

// buffer index of stored element e: Neumann x_e = node e; hinged x_{e+1} = interior node e+1
template <int NEUMANN>
PD_DEV int bidx(int e) { return NEUMANN ? e : e + 1; }

// y_j from x_j and x_{M-j}
template <int NEUMANN>
PD_DEV double ymap(double xj, double xm, double s) {
  return NEUMANN ? 0.5 * (xj + xm) - s * (xj - xm) : s * (xj + xm) + 0.5 * (xj - xm);
}

// In-place pre-processing of one line held in xb (double view, dpad layout, x_0..x_M present;
// hinged lines carry explicit zeros at 0 and M).  Pairs (n, H-1-n) are processed in phases of 32
// consecutive n: every lane reads its six inputs, the warp syncs, then writes; the single value a
// phase needs from the previous one (x_{M-2n} for its first pair) is carried from lane 31.
// Returns X_1 (DCT-I) summed over the warp, 0 for DST-I.
template <int NEUMANN>
PD_DEV double dtt_pre(double* xb, int M, const double2* __restrict__ trig, int lane) {
  const int NP = M >> 2;                 // pairs
  double x1 = 0.0, carry = 0.0;
  for (int base = 0; base < NP; base += 32) {
    const int n = base + lane;
    const bool act = n < NP;
    double A = 0, B = 0, C = 0, D = 0, E = 0, F = 0;
    if (act) {
      A = xb[dpad(2 * n)];
      B = xb[dpad(2 * n + 1)];
      C = xb[dpad(2 * n + 2)];
      D = xb[dpad(M - 2 * n - 2)];
      E = xb[dpad(M - 2 * n - 1)];
      F = (lane == 0 && base > 0) ? carry : xb[dpad(M - 2 * n)];
    }
    carry = __shfl_sync(0xffffffffu, D, 31);
    __syncwarp();
    if (act) {
      const int j0 = 2 * n, j1 = 2 * n + 1, j2 = M - 2 * n - 2, j3 = M - 2 * n - 1;
      const double2 t0 = __ldg(trig + j0), t1 = __ldg(trig + j1), t2 = __ldg(trig + j2), t3 = __ldg(trig + j3);
      xb[dpad(j0)] = ymap<NEUMANN>(A, F, t0.y);
      xb[dpad(j1)] = ymap<NEUMANN>(B, E, t1.y);
      xb[dpad(j2)] = ymap<NEUMANN>(D, C, t2.y);
      xb[dpad(j3)] = ymap<NEUMANN>(E, B, t3.y);
      if (NEUMANN) x1 += ((A - F) * t0.x + (B - E) * t1.x) + ((D - C) * t2.x + (E - B) * t3.x);
    }
    __syncwarp();
  }
  return NEUMANN ? warp_sum(x1) : 0.0;
}

// Post-processing: for k-chunks of 32 (lane = k - k0) emit the outputs through
// `emit(idx, value, k0)` (idx = stored element index along the line) and call `chunk_end(k0)`
// after each chunk.  Chunk k0 emits stored indices within [2k0 - 1, 2k0 + 64].
template <int NEUMANN, class Emit, class ChunkEnd>
PD_DEV void dtt_post(const double2* zb, int M, int log2h, double x1, const double2* __restrict__ trig,
                     int lane, Emit emit, ChunkEnd chunk_end) {
  const int H = M >> 1;
  double carry = 0.0;
  for (int k0 = 0; k0 < H; k0 += 32) {
    const int k = k0 + lane;
    double ev = 0.0, scanv = 0.0;
    if (k < H) {
      const double2 Zk = zb[pad16(bitrev(k, log2h))];
      const double2 Zm = zb[pad16(bitrev((H - k) & (H - 1), log2h))];
      const double2 E = make_double2(0.5 * (Zk.x + Zm.x), 0.5 * (Zk.y - Zm.y));
      const double2 O = make_double2(0.5 * (Zk.y + Zm.y), -0.5 * (Zk.x - Zm.x));
      const double2 t2 = __ldg(trig + 2 * k);            // W_M^k = cos - i sin
      const double2 Y = make_double2(E.x + t2.x * O.x + t2.y * O.y, E.y + t2.x * O.y - t2.y * O.x);
      if (NEUMANN) {
        ev = 2.0 * Y.x;
        scanv = k == 0 ? 0.0 : Y.y;
      } else {
        ev = -2.0 * Y.y;
        scanv = k == 0 ? Y.x : 2.0 * Y.x;
      }
    }
    double incl = scanv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const double S = carry + incl;
    carry += __shfl_sync(0xffffffffu, incl, 31);
    if (k < H) {
      if (NEUMANN) {
        emit(2 * k, ev, k0);                 // X_{2k}
        emit(2 * k + 1, x1 - 2.0 * S, k0);   // X_{2k+1}
      } else {
        emit(2 * k, S, k0);                  // X_{2k+1} (stored index 2k)
        if (k > 0) emit(2 * k - 1, ev, k0);  // X_{2k}   (stored index 2k-1)
      }
    }
    if (NEUMANN && k0 + 32 >= H && lane == 0) {
      const double2 Z0 = zb[pad16(0)];
      emit(M, 2.0 * (Z0.x - Z0.y), k0);      // X_M = 2 Re Y_{M/2}
    }
    chunk_end(k0);
  }
}

// ---------------------------------------------------------------- rows (x axis)
template <int NEUMANN, int NW>
__global__ void __launch_bounds__(NW * 32)
k_dtt_rows(const double* in, double* out, LineParams P) {
  extern __shared__ double2 smem2[];
  double* xb = reinterpret_cast<double*>(smem2) + (size_t)(threadIdx.x >> 5) * dpadded(P.M);
  const int lane = threadIdx.x & 31;
  const int M = P.M;
  double lmax = 0.0;
  for (int64_t L = (int64_t)blockIdx.x * NW + (threadIdx.x >> 5); L < P.nlines; L += (int64_t)gridDim.x * NW) {
    const double* src = in + L * P.nx;
    double* dst = out + L * P.nx;
    for (int e = lane; e < P.nel; e += 32) cp_async8(xb + dpad(bidx<NEUMANN>(e)), src + e);
    cp_async_commit();
    if (!NEUMANN && lane == 0) {
      xb[dpad(0)] = 0.0;
      xb[dpad(M)] = 0.0;
    }
    cp_async_wait_all();
    __syncwarp();
    const double x1 = dtt_pre<NEUMANN>(xb, M, P.trig, lane);
    double2* zb = reinterpret_cast<double2*>(xb);
    warp_fft_dif<-1>(zb, P.log2h, P.tw, P.twlog, lane);
    dtt_post<NEUMANN>(zb, M, P.log2h, x1, P.trig, lane,
                      [&](int idx, double v, int) {
                        dst[idx] = v;
                        lmax = fmax(lmax, fabs(v));
                      },
                      [](int) {});
    __syncwarp();
  }
  if (P.amax) warp_atomic_max_abs(P.amax, lmax);
}

// ---------------------------------------------------------------- columns (y axis)
// CTA = W warps on W adjacent columns of one slice; rows are loaded W doubles at a time.
template <int NEUMANN, int W>
__global__ void __launch_bounds__(W * 32)
k_dtt_cols(const double* in, double* out, LineParams P) {
  extern __shared__ double2 smem2[];
  double* base = reinterpret_cast<double*>(smem2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = P.M;
  const int LD = dpadded(M);
  double* xb = base + (size_t)warp * LD;
  double* stage = base + (size_t)W * LD;                 // [66][W] output staging
  const int64_t gx = (P.nx + W - 1) / W;
  const int64_t ngroups = (P.nlines / P.nx) * gx;
  double lmax = 0.0;
  for (int64_t G = blockIdx.x; G < ngroups; G += gridDim.x) {
    const int64_t n = G / gx;
    const int x0 = (int)((G - n * gx) * W);
    const double* src = in + n * P.ns + x0;
    double* dst = out + n * P.ns + x0;
    const int wcols = min(W, (int)(P.nx - x0));
    for (int idx = threadIdx.x; idx < P.nel * W; idx += W * 32) {
      const int e = idx / W, c = idx - e * W;
      if (c < wcols) cp_async8(base + (size_t)c * LD + dpad(bidx<NEUMANN>(e)), src + (int64_t)e * P.nx + c);
    }
    cp_async_commit();
    if (!NEUMANN && lane == 0) {
      xb[dpad(0)] = 0.0;
      xb[dpad(M)] = 0.0;
    }
    cp_async_wait_all();
    __syncthreads();
    const bool live = warp < wcols;
    double x1 = 0.0;
    double2* zb = reinterpret_cast<double2*>(xb);
    if (live) {
      x1 = dtt_pre<NEUMANN>(xb, M, P.trig, lane);
      warp_fft_dif<-1>(zb, P.log2h, P.tw, P.twlog, lane);
    }
    // chunk k0 emits stored indices [2k0 - 1, 2k0 + 64] -> staging row idx - 2k0 + 1 (66 rows)
    const int H = M >> 1;
    dtt_post<NEUMANN>(zb, M, P.log2h, x1, P.trig, lane,
                      [&](int idx, double v, int k0) {
                        if (live) stage[(idx - 2 * k0 + 1) * W + warp] = v;
                      },
                      [&](int k0) {
                        __syncthreads();
                        int lo, hi;
                        if (NEUMANN) {
                          lo = 2 * k0;
                          hi = k0 + 32 >= H ? M + 1 : 2 * (k0 + 32);
                        } else {
                          lo = max(2 * k0 - 1, 0);
                          hi = min(2 * k0 + 63, P.nel);
                        }
                        for (int i = threadIdx.x; i < (hi - lo) * W; i += W * 32) {
                          const int r = i / W, c = i - r * W;
                          if (c < wcols) {
                            const double v = stage[(lo + r - 2 * k0 + 1) * W + c];
                            dst[(int64_t)(lo + r) * P.nx + c] = v;
                            lmax = fmax(lmax, fabs(v));
                          }
                        }
                        __syncthreads();
                      });
  }
  if (P.amax) warp_atomic_max_abs(P.amax, lmax);
}

}  // namespace pd
