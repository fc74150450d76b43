// shard.cu — the multi-rank ParaDiag iteration behind the C ABI.
//
// Why it shards ("Step-(2) is fully parallel"): the preconditioner is three commuting
// transforms — x, y (DCT-I / DST-I) and time (Γ_α·DFT) — around a per-mode
// divide.  Rank r of P owns
//   * the ROW slab y ∈ rows[r] of every time slice: residual (a 2-row halo from each
//     neighbour), forward / inverse x transforms, update;
//   * the COLUMN slab x ∈ cols[r] (x-modes after the x transform): y transforms and the time pass —
//     every local point has its whole time pencil, so Step (2) needs no communication.
// Two all-to-alls per P_α⁻¹ move the (row slab r) × (column slab q) blocks between the layouts;
// the passes next to them read and write the transpose blocks directly (paradiag_slab_*_seg, no
// pack / unpack copies), and the block a rank keeps stays in a private region (never sent).  The
// stop rule's ‖δ‖∞ / ‖U‖∞ are max-all-reduced.  The library owns the NCCL communicator: rank 0
// draws the 128-byte id (paradiag_nccl_unique_id), the caller broadcasts it, every rank calls
// paradiag_init(…, id, rank, nranks).  NCCL is resolved at run time from the copy the process has
// already loaded (torch's), so one process never holds two NCCLs.
//
// The same orchestration drives VIRTUAL ranks: P slab handles in one process on one device, the
// collectives emulated by device copies in rank order (no rank ever waits on another, which
// B200_PROFILING.md requires when ranks share a GPU) — the test of the layout and the block
// addressing without a multi-GPU box.
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "nccl.h"
#include "shard.h"

namespace {

// ---------------------------------------------------------------- NCCL, resolved at run time
struct Nccl {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  bool ok = false;
};

const Nccl* nccl() {
  static Nccl api;
  static bool tried = false;
  if (tried) return api.ok ? &api : nullptr;
  tried = true;
  // the NCCL already in the process (torch links it), else whatever the loader finds
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return nullptr;
#define PD_SYM(f, n) api.f = reinterpret_cast<decltype(api.f)>(dlsym(lib, n))
  PD_SYM(getUniqueId, "ncclGetUniqueId");
  PD_SYM(commInitRank, "ncclCommInitRank");
  PD_SYM(commDestroy, "ncclCommDestroy");
  PD_SYM(allReduce, "ncclAllReduce");
  PD_SYM(send, "ncclSend");
  PD_SYM(recv, "ncclRecv");
  PD_SYM(groupStart, "ncclGroupStart");
  PD_SYM(groupEnd, "ncclGroupEnd");
  PD_SYM(errorString, "ncclGetErrorString");
#undef PD_SYM
  api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce && api.send && api.recv &&
           api.groupStart && api.groupEnd && api.errorString;
  return api.ok ? &api : nullptr;
}

int nccl_fail(ncclResult_t r, const char* what) {
  const Nccl* n = nccl();
  std::string m = std::string(what) + ": " + (n ? n->errorString(r) : "NCCL");
  return pd_set_error(PD_ENCCL, m.c_str());
}

#define PD_NCCL(call)                                           \
  do {                                                          \
    ncclResult_t r_ = (call);                                   \
    if (r_ != ncclSuccess) return nccl_fail(r_, #call);         \
  } while (0)

#define PD_CHECK(call)                                          \
  do {                                                          \
    int rc_ = (call);                                           \
    if (rc_ < 0) return rc_;                                    \
  } while (0)

#define PD_CU(call)                                                                                     \
  do {                                                                                                 \
    cudaError_t e_ = (call);                                                                           \
    if (e_ != cudaSuccess) return pd_set_error(e_ == cudaErrorMemoryAllocation ? PD_ENOMEM : PD_ECUDA, \
                                               (std::string(#call) + ": " + cudaGetErrorString(e_)).c_str()); \
  } while (0)

std::vector<std::pair<int64_t, int64_t>> split(int64_t n, int parts) {   // (start, count) per part
  std::vector<std::pair<int64_t, int64_t>> out;
  const int64_t base = n / parts, extra = n % parts;
  int64_t s = 0;
  for (int p = 0; p < parts; ++p) {
    const int64_t c = base + (p < extra ? 1 : 0);
    out.push_back({s, c});
    s += c;
  }
  return out;
}

struct Group {                      // the ranks this process drives: one (NCCL) or all (virtual)
  int P = 1;
  bool virt = false;
  ncclComm_t comm = nullptr;
  std::vector<pd_handle*> hs;       // virtual: every rank's handle, in rank order
  int refs = 0;
};

}  // namespace

struct pd_shard {
  Group* g = nullptr;
  int rank = 0;
  int64_t n = 0, nt = 0, y0 = 0, nyl = 0, x0 = 0, nxl = 0;
  int64_t nsr = 0, so = 0, hs = 0;
  std::vector<int64_t> fs, fr, cfs, cfr;                 // forward send / receive splits and offsets
  std::vector<int64_t> xm_out, ym_in, ym_out, xm_in;     // transpose-block maps {k, (e0, cnt, off) × k}
  std::vector<void*> allocs;
  double* rowsb = nullptr;   // r, then δ on the row slab [nt][nyl][n]
  double* cols = nullptr;    // column slab [nt][n][nxl]
  double* buf = nullptr;     // [send | recv | self] transpose blocks
  double *hsl = nullptr, *hsh = nullptr, *hlo = nullptr, *hhi = nullptr;   // halo send lo/hi, recv lo/hi
  double* u0buf = nullptr;   // window hand-off [nyl][n]
  pd_problem P{};
};

namespace {

int salloc(pd_shard* s, double** p, int64_t count) {
  void* q = nullptr;
  PD_CU(cudaMalloc(&q, (size_t)std::max<int64_t>(count, 1) * sizeof(double)));
  s->allocs.push_back(q);
  *p = static_cast<double*>(q);
  return PD_OK;
}

// layout of rank r (the fused, single-range form of dist.SlabRank)
void layout(pd_shard* s, int P, int r) {
  const auto rows = split(s->n, P), cols = split(s->n, P);
  s->y0 = rows[r].first;
  s->nyl = rows[r].second;
  s->x0 = cols[r].first;
  s->nxl = cols[r].second;
  s->fs.assign(P, 0);
  s->fr.assign(P, 0);
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    s->fs[q] = s->nt * s->nyl * cols[q].second;
    s->fr[q] = s->nt * rows[q].second * s->nxl;
  }
  int64_t a = 0, b = 0;
  s->cfs.assign(P, 0);
  s->cfr.assign(P, 0);
  for (int q = 0; q < P; ++q) {
    s->cfs[q] = a;
    s->cfr[q] = b;
    a += s->fs[q];
    b += s->fr[q];
  }
  s->nsr = std::max(a, b);
  s->so = 2 * s->nsr;
  auto map = [&](const std::vector<std::pair<int64_t, int64_t>>& sp, int64_t base, const std::vector<int64_t>& cum) {
    std::vector<int64_t> m{(int64_t)P};
    for (int q = 0; q < P; ++q) {
      m.push_back(sp[q].first);
      m.push_back(sp[q].second);
      m.push_back(q == r ? s->so : base + cum[q]);
    }
    return m;
  };
  s->xm_out = map(cols, 0, s->cfs);
  s->ym_in = map(rows, s->nsr, s->cfr);
  s->ym_out = map(rows, 0, s->cfr);
  s->xm_in = map(cols, s->nsr, s->cfs);
  s->hs = s->nt * 2 * s->n;
}

int make_shard(pd_handle* h, const pd_problem* p, Group* g, int r) {
  pd_shard* s = new pd_shard;
  s->P = *p;
  s->g = g;
  s->rank = r;
  const int64_t n = p->bc == PD_BC_NEUMANN ? p->m + 1 : p->m - 1;
  s->n = n;
  s->nt = p->nt;
  layout(s, g->P, r);
  pd_handle_shard(h) = s;
  g->refs += 1;
  PD_CHECK(salloc(s, &s->rowsb, s->nt * s->nyl * n));
  PD_CHECK(salloc(s, &s->cols, s->nt * n * s->nxl));
  PD_CHECK(salloc(s, &s->buf, s->so + s->nt * s->nyl * s->nxl));
  PD_CHECK(salloc(s, &s->u0buf, s->nyl * n));
  if (g->P > 1) {
    PD_CHECK(salloc(s, &s->hsl, s->hs));
    PD_CHECK(salloc(s, &s->hsh, s->hs));
    if (r > 0) PD_CHECK(salloc(s, &s->hlo, s->hs));
    if (r < g->P - 1) PD_CHECK(salloc(s, &s->hhi, s->hs));
  }
  return PD_OK;
}

int check_problem(const pd_problem* p, int nranks) {
  if (!p) return pd_set_error(PD_EINVAL, "problem is NULL");
  if (nranks < 1 || nranks > 8) return pd_set_error(PD_EINVAL, "sharded: 1 <= nranks <= 8 (transpose-block maps)");
  if (p->dim != 2 || !(p->kind == PD_BIHARMONIC || p->kind == PD_LINEAR_CH) || p->theta != 1.0 ||
      p->jacobian != PD_JACOBIAN_SCALAR)
    return pd_set_error(PD_EINVAL, "sharded: 2D linear kinds with theta = 1 (CH runs as replicas, DESIGN.md §8)");
  const int64_t n = p->bc == PD_BC_NEUMANN ? p->m + 1 : p->m - 1;
  if (n / nranks < 3) return pd_set_error(PD_EINVAL, "sharded: at least 3 rows per rank");
  return PD_OK;
}

// ---------------------------------------------------------------- collectives (group-wide)
pd_shard* S(pd_handle* h) { return pd_handle_shard(h); }

struct NvtxRange {                    // NVTX range of a collective (C1-C3)
  explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
  ~NvtxRange() { nvtxRangePop(); }
};

int comm_halo(Group* g) {
  if (g->P == 1) return PD_OK;
  NvtxRange nv("halo_exchange");
  if (g->virt) {                     // rank r's first rows -> r-1's upper halo, last rows -> r+1's lower halo
    for (int r = 0; r < g->P; ++r) {
      pd_shard* s = S(g->hs[r]);
      const cudaStream_t st = pd_handle_stream(g->hs[r]);
      if (r > 0) PD_CU(cudaMemcpyAsync(S(g->hs[r - 1])->hhi, s->hsl, s->hs * 8, cudaMemcpyDeviceToDevice, st));
      if (r < g->P - 1) PD_CU(cudaMemcpyAsync(S(g->hs[r + 1])->hlo, s->hsh, s->hs * 8, cudaMemcpyDeviceToDevice, st));
    }
    return PD_OK;
  }
  const Nccl* N = nccl();
  pd_handle* h = g->hs[0];
  pd_shard* s = S(h);
  const cudaStream_t st = pd_handle_stream(h);
  const int r = s->rank;
  PD_NCCL(N->groupStart());
  if (r > 0) {
    PD_NCCL(N->send(s->hsl, s->hs, ncclFloat64, r - 1, g->comm, st));
    PD_NCCL(N->recv(s->hlo, s->hs, ncclFloat64, r - 1, g->comm, st));
  }
  if (r < g->P - 1) {
    PD_NCCL(N->send(s->hsh, s->hs, ncclFloat64, r + 1, g->comm, st));
    PD_NCCL(N->recv(s->hhi, s->hs, ncclFloat64, r + 1, g->comm, st));
  }
  PD_NCCL(N->groupEnd());
  return PD_OK;
}

// dir 0: forward (rows -> columns), 1: backward.  Sends from [0, nsr), receives into [nsr, 2 nsr).
int comm_a2a(Group* g, int dir) {
  if (g->P == 1) return PD_OK;
  NvtxRange nv(dir == 0 ? "alltoall_fwd" : "alltoall_bwd");
  if (g->virt) {
    for (int r = 0; r < g->P; ++r) {
      pd_shard* s = S(g->hs[r]);
      const cudaStream_t st = pd_handle_stream(g->hs[r]);
      for (int q = 0; q < g->P; ++q) {
        if (q == r) continue;
        pd_shard* t = S(g->hs[q]);
        const int64_t cnt = dir == 0 ? s->fs[q] : s->fr[q];
        const int64_t soff = dir == 0 ? s->cfs[q] : s->cfr[q];
        const int64_t roff = t->nsr + (dir == 0 ? t->cfr[r] : t->cfs[r]);
        PD_CU(cudaMemcpyAsync(t->buf + roff, s->buf + soff, cnt * 8, cudaMemcpyDeviceToDevice, st));
      }
    }
    return PD_OK;
  }
  const Nccl* N = nccl();
  pd_handle* h = g->hs[0];
  pd_shard* s = S(h);
  const cudaStream_t st = pd_handle_stream(h);
  PD_NCCL(N->groupStart());
  for (int q = 0; q < g->P; ++q) {
    if (q == s->rank) continue;
    const int64_t scnt = dir == 0 ? s->fs[q] : s->fr[q], soff = dir == 0 ? s->cfs[q] : s->cfr[q];
    const int64_t rcnt = dir == 0 ? s->fr[q] : s->fs[q], roff = s->nsr + (dir == 0 ? s->cfr[q] : s->cfs[q]);
    PD_NCCL(N->send(s->buf + soff, scnt, ncclFloat64, q, g->comm, st));
    PD_NCCL(N->recv(s->buf + roff, rcnt, ncclFloat64, q, g->comm, st));
  }
  PD_NCCL(N->groupEnd());
  return PD_OK;
}

// global (‖δ‖∞, ‖U‖∞): max over the ranks of the handles' statistics (bit-pattern maxima)
int comm_stats(Group* g, double* dmax, double* umax) {
  NvtxRange nv("allreduce_stats");
  if (!g->virt && g->comm)          // (a one-rank world runs it too: the NCCL path is exercised)
    PD_NCCL(nccl()->allReduce(pd_handle_stats_dev(g->hs[0]), pd_handle_stats_dev(g->hs[0]), 2, ncclUint64, ncclMax,
                              g->comm, pd_handle_stream(g->hs[0])));
  *dmax = 0.0;
  *umax = 0.0;
  for (pd_handle* h : g->hs) {
    double d, u;
    PD_CHECK(paradiag_stats_read(h, &d, &u));
    if (!(d <= *dmax)) *dmax = d;                       // NaN propagates (never <=)
    if (!(u <= *umax)) *umax = u;
  }
  return PD_OK;
}

// ---------------------------------------------------------------- one iteration / P_α⁻¹, group-wide
int group_precond(Group* g, const double* const* r, double* const* delta, int want_dmax) {
  for (int k = 0; k < (int)g->hs.size(); ++k) {
    pd_shard* s = S(g->hs[k]);
    PD_CHECK(paradiag_slab_xpass_seg(g->hs[k], r[k], s->buf, 0, nullptr, s->xm_out.data()));
  }
  PD_CHECK(comm_a2a(g, 0));
  for (pd_handle* h : g->hs) {
    pd_shard* s = S(h);
    PD_CHECK(paradiag_slab_ypass_seg(h, s->buf, s->cols, s->buf, s->ym_in.data(), s->ym_out.data()));
  }
  PD_CHECK(comm_a2a(g, 1));
  for (int k = 0; k < (int)g->hs.size(); ++k) {
    pd_shard* s = S(g->hs[k]);
    PD_CHECK(paradiag_slab_xpass_seg(g->hs[k], s->buf, delta[k], want_dmax, s->xm_in.data(), nullptr));
  }
  return PD_OK;
}

int group_iterate(Group* g, const double* const* u0, double* const* U, double* dmax, double* umax) {
  const int L = (int)g->hs.size();
  for (int k = 0; k < L; ++k) {
    pd_handle* h = g->hs[k];
    pd_shard* s = S(h);
    PD_CHECK(paradiag_stats_reset(h));
    if (g->P > 1) {                // halo packs: rows {0, 1} and {nyl-2, nyl-1} of every slice
      PD_CHECK(paradiag_copy3d(h, U[k], s->hsl, s->nt, 2, s->n, s->nyl * s->n, s->n, 2 * s->n, s->n));
      PD_CHECK(paradiag_copy3d(h, U[k] + (s->nyl - 2) * s->n, s->hsh, s->nt, 2, s->n, s->nyl * s->n, s->n, 2 * s->n,
                               s->n));
    }
  }
  PD_CHECK(comm_halo(g));
  std::vector<const double*> rr(L);
  std::vector<double*> dd(L);
  for (int k = 0; k < L; ++k) {
    pd_shard* s = S(g->hs[k]);
    PD_CHECK(paradiag_slab_residual(g->hs[k], u0[k], U[k], s->hlo, s->hhi, s->rowsb));
    rr[k] = s->rowsb;
    dd[k] = s->rowsb;
  }
  PD_CHECK(group_precond(g, rr.data(), dd.data(), 1));
  for (int k = 0; k < L; ++k) PD_CHECK(paradiag_slab_update(g->hs[k], U[k], S(g->hs[k])->rowsb));
  return comm_stats(g, dmax, umax);
}

int group_init_iterate(Group* g, const double* const* u0, double* const* U) {
  for (int k = 0; k < (int)g->hs.size(); ++k) {
    pd_shard* s = S(g->hs[k]);
    const cudaStream_t st = pd_handle_stream(g->hs[k]);
    if (s->P.init == PD_INIT_ZERO) {
      PD_CU(cudaMemsetAsync(U[k], 0, (size_t)s->nt * s->nyl * s->n * 8, st));
    } else {                         // U⁰ = u0 broadcast to every slice (R#5): a stride-0 copy
      PD_CHECK(paradiag_copy3d(g->hs[k], u0[k], U[k], s->nt, s->nyl, s->n, 0, s->n, s->nyl * s->n, s->n));
    }
  }
  return PD_OK;
}

int group_solve(Group* g, const double* const* u0_in, double* const* U, pd_solve_info* info) {
  const pd_problem& p = S(g->hs[0])->P;
  const int L = (int)g->hs.size();
  std::memset(info, 0, sizeof(*info));
  std::vector<const double*> u0(u0_in, u0_in + L);
  int status = PD_OK;
  bool all_conv = true;
  for (int w = 0; w < p.n_windows; ++w) {
    PD_CHECK(group_init_iterate(g, u0.data(), U));
    const int kmax = p.fixed_iters > 0 ? p.fixed_iters : p.max_iter;
    bool conv = false, div = false;
    int k = 0, growth = 0;
    double dprev = 0.0, dmax = 0.0, umax = 0.0;
    for (k = 1; k <= kmax; ++k) {
      PD_CHECK(group_iterate(g, u0.data(), U, &dmax, &umax));
      if (!(dmax == dmax) || !(umax == umax) || dmax > 1.7e308 || umax > 1.7e308) {
        info->iters[w] = k;
        info->windows_done = w;
        return pd_set_error(PD_EDIVERGED, "non-finite increment or iterate");
      }
      if (p.fixed_iters <= 0 && dmax <= p.tol * umax) {
        conv = true;
        break;
      }
      growth = (k > 1 && dmax > dprev) ? growth + 1 : 0;              // SURVEY §5.3 (PD_GROWTH_LIMIT)
      dprev = dmax;
      if (growth >= PD_GROWTH_LIMIT) {
        div = true;
        if (p.fixed_iters <= 0) break;
      }
    }
    info->iters[w] = std::min(k, kmax);
    info->last_rel[w] = umax > 0 ? dmax / umax : 0.0;
    info->diverging += div ? 1 : 0;
    info->windows_done = w + 1;
    all_conv = all_conv && conv;
    if (!conv && p.fixed_iters <= 0) status = PD_NOT_CONVERGED;
    if (w + 1 < p.n_windows) {       // hand-off u0 <- U_{N_t}: each rank its own rows
      for (int j = 0; j < L; ++j) {
        pd_shard* s = S(g->hs[j]);
        PD_CU(cudaMemcpyAsync(s->u0buf, U[j] + (s->nt - 1) * s->nyl * s->n, s->nyl * s->n * 8,
                              cudaMemcpyDeviceToDevice, pd_handle_stream(g->hs[j])));
        u0[j] = s->u0buf;
      }
    }
  }
  info->converged = p.fixed_iters > 0 ? 0 : (all_conv ? 1 : 0);
  for (pd_handle* h : g->hs) PD_CU(cudaStreamSynchronize(pd_handle_stream(h)));
  return status;
}

Group* own_group(pd_handle* h) {      // an NCCL rank's group holds just its own handle
  pd_shard* s = S(h);
  return s ? s->g : nullptr;
}

}  // namespace

// ---------------------------------------------------------------- internal entry points
int shard_unique_id(unsigned char id[128]) {
  if (!id) return pd_set_error(PD_EINVAL, "id is NULL");
  const Nccl* N = nccl();
  if (!N) return pd_set_error(PD_ENCCL, "libnccl.so.2 not found (import torch first: the library uses its NCCL)");
  ncclUniqueId u;
  PD_NCCL(N->getUniqueId(&u));
  std::memcpy(id, u.internal, 128);
  return PD_OK;
}

int shard_init(const pd_problem* p, int device, void* cuda_stream, const unsigned char* nccl_id, int rank,
               int nranks, pd_handle** out) {
  if (!out) return pd_set_error(PD_EINVAL, "out is NULL");
  *out = nullptr;
  PD_CHECK(check_problem(p, nranks));
  if (rank < 0 || rank >= nranks) return pd_set_error(PD_EINVAL, "rank outside [0, nranks)");
  const int64_t n = p->bc == PD_BC_NEUMANN ? p->m + 1 : p->m - 1;
  const auto rows = split(n, nranks), cols = split(n, nranks);
  pd_handle* h = nullptr;
  PD_CHECK(paradiag_init_slab(p, device, cuda_stream, rows[rank].first, rows[rank].second, cols[rank].first,
                              cols[rank].second, &h));
  Group* g = new Group;
  g->P = nranks;
  g->hs = {h};
  int rc = make_shard(h, p, g, rank);
  if (rc == PD_OK && nccl_id) {
    const Nccl* N = nccl();
    if (!N) {
      rc = pd_set_error(PD_ENCCL, "libnccl.so.2 not found (import torch first: the library uses its NCCL)");
    } else {
      ncclUniqueId u;
      std::memcpy(u.internal, nccl_id, 128);
      cudaSetDevice(device);
      const ncclResult_t r = N->commInitRank(&g->comm, nranks, u, rank);
      if (r != ncclSuccess) rc = nccl_fail(r, "ncclCommInitRank");
    }
  } else if (rc == PD_OK && nranks > 1) {
    rc = pd_set_error(PD_EINVAL, "nranks > 1 needs an NCCL id (paradiag_nccl_unique_id on rank 0)");
  }
  if (rc) {
    paradiag_destroy(h);
    return rc;
  }
  *out = h;
  return PD_OK;
}

int shard_apply_precond(pd_handle* h, const double* r, double* delta) {
  Group* g = own_group(h);
  return group_precond(g, &r, &delta, 0);
}

int shard_iterate(pd_handle* h, const double* u0_l, double* U_l, pd_iter_info* info) {
  Group* g = own_group(h);
  double dmax = 0, umax = 0;
  pd_iter_info tmp = *info;
  PD_CHECK(group_iterate(g, &u0_l, &U_l, &dmax, &umax));
  tmp.iters = info->iters + 1;
  tmp.delta_max = dmax;
  tmp.u_max = umax;
  tmp.rel = umax > 0 ? dmax / umax : 0.0;
  tmp.jbar = 0.0;
  tmp.omega = 1.0;
  tmp.converged = S(h)->P.fixed_iters <= 0 && dmax <= S(h)->P.tol * umax;
  tmp.growth = (info->iters > 0 && dmax > info->delta_max) ? info->growth + 1 : 0;
  *info = tmp;
  if (!(dmax == dmax) || !(umax == umax) || dmax > 1.7e308 || umax > 1.7e308)
    return pd_set_error(PD_EDIVERGED, "non-finite increment or iterate");
  return PD_OK;
}

int shard_solve(pd_handle* h, const double* u0_l, double* U_l, pd_solve_info* info) {
  return group_solve(own_group(h), &u0_l, &U_l, info);
}

int shard_local_rows(const pd_handle* h, int64_t* y0, int64_t* nyl) {
  pd_shard* s = pd_handle_shard(const_cast<pd_handle*>(h));
  if (y0) *y0 = s->y0;
  if (nyl) *nyl = s->nyl;
  return PD_OK;
}

void shard_destroy(pd_shard* s) {
  if (!s) return;
  for (void* q : s->allocs) cudaFree(q);
  Group* g = s->g;
  delete s;
  if (g && --g->refs <= 0) {
    if (g->comm && nccl()) nccl()->commDestroy(g->comm);
    delete g;
  }
}

// ---------------------------------------------------------------- public: virtual ranks
int paradiag_init_virtual(const pd_problem* p, int device, void* cuda_stream, int nranks, pd_handle** out) {
  if (!out) return pd_set_error(PD_EINVAL, "out is NULL");
  PD_CHECK(check_problem(p, nranks));
  const int64_t n = p->bc == PD_BC_NEUMANN ? p->m + 1 : p->m - 1;
  const auto rows = split(n, nranks), cols = split(n, nranks);
  Group* g = new Group;
  g->P = nranks;
  g->virt = true;
  for (int r = 0; r < nranks; ++r) out[r] = nullptr;
  for (int r = 0; r < nranks; ++r) {
    pd_handle* h = nullptr;
    int rc = paradiag_init_slab(p, device, cuda_stream, rows[r].first, rows[r].second, cols[r].first,
                                cols[r].second, &h);
    if (rc == PD_OK) {
      g->hs.push_back(h);
      out[r] = h;
      rc = make_shard(h, p, g, r);
    }
    if (rc) {
      for (int q = 0; q <= r; ++q)
        if (out[q]) paradiag_destroy(out[q]);
      if (g->refs == 0) delete g;
      return rc;
    }
  }
  return PD_OK;
}

static int virtual_group(pd_handle* const* hs, int nranks, Group** g) {
  if (!hs || nranks < 1 || !hs[0] || !pd_handle_shard(hs[0])) return pd_set_error(PD_EINVAL, "not virtual ranks");
  *g = pd_handle_shard(hs[0])->g;
  if (!(*g)->virt || (*g)->P != nranks) return pd_set_error(PD_EINVAL, "handles are not one virtual group");
  for (int r = 0; r < nranks; ++r)
    if (hs[r] != (*g)->hs[r]) return pd_set_error(PD_EINVAL, "handles out of rank order");
  return PD_OK;
}

int paradiag_iterate_virtual(pd_handle* const* hs, int nranks, const double* const* u0_l, double* const* U_l,
                             pd_iter_info* info) {
  Group* g = nullptr;
  PD_CHECK(virtual_group(hs, nranks, &g));
  if (!u0_l || !U_l || !info) return pd_set_error(PD_EINVAL, "NULL argument");
  double dmax = 0, umax = 0;
  PD_CHECK(group_iterate(g, u0_l, U_l, &dmax, &umax));
  pd_iter_info tmp = *info;
  tmp.iters = info->iters + 1;
  tmp.delta_max = dmax;
  tmp.u_max = umax;
  tmp.rel = umax > 0 ? dmax / umax : 0.0;
  tmp.omega = 1.0;
  tmp.converged = S(hs[0])->P.fixed_iters <= 0 && dmax <= S(hs[0])->P.tol * umax;
  tmp.growth = (info->iters > 0 && dmax > info->delta_max) ? info->growth + 1 : 0;
  *info = tmp;
  return PD_OK;
}

int paradiag_solve_virtual(pd_handle* const* hs, int nranks, const double* const* u0_l, double* const* U_l,
                           pd_solve_info* info) {
  Group* g = nullptr;
  PD_CHECK(virtual_group(hs, nranks, &g));
  if (!u0_l || !U_l || !info) return pd_set_error(PD_EINVAL, "NULL argument");
  return group_solve(g, u0_l, U_l, info);
}

// ---------------------------------------------------------------- public: the layout (host only)
int paradiag_shard_layout(int64_t n, int64_t nt, int nranks, int rank, int64_t* out, int64_t cap) {
  if (!out || nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks || n / nranks < 3 || nt < 1)
    return pd_set_error(PD_EINVAL, "shard layout: bad arguments");
  const int64_t P = nranks, need = 6 + 4 * P + 4 * (1 + 3 * P);
  if (cap < need) return pd_set_error(PD_EINVAL, "shard layout: output too small");
  pd_shard s;
  s.n = n;
  s.nt = nt;
  layout(&s, nranks, rank);
  int64_t k = 0;
  for (int64_t v : {s.y0, s.nyl, s.x0, s.nxl, s.nsr, s.so}) out[k++] = v;
  for (const auto* v : {&s.fs, &s.fr, &s.cfs, &s.cfr})
    for (int64_t x : *v) out[k++] = x;
  for (const auto* v : {&s.xm_out, &s.ym_in, &s.ym_out, &s.xm_in})
    for (int64_t x : *v) out[k++] = x;
  return PD_OK;
}
