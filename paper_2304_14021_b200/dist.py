"""Multi-rank ParaDiag iteration: one process per GPU, the 2D grid sharded in slabs (SURVEY §8(e),
DESIGN.md §8).

Why it shards ("Step-(2) is fully parallel"): the preconditioner is three commuting
transforms — x, y (DCT-I / DST-I) and time (Γ_α·DFT) — with a per-mode divide
in the middle.  Each rank r owns

  * the ROW slab  y ∈ rows[r] of every time slice: residual (needs a 2-row halo from
    the neighbouring ranks), x transforms, update;
  * the COLUMN slab x ∈ cols[r] (x-modes after the x transform): y transforms and the time pass
    (complete time pencils of every local point, so Step-(2) needs no further communication).

Between the layouts an all-to-all transposes the data (forward after the x transform, backward
before the inverse x transform).  The collectives are torch.distributed (NCCL on GPUs, gloo in
the CPU tests); every local step runs in the C-ABI library (slab entry points of
include/paradiag.h) through ``GpuOps``.  The copy descriptors of the packs / unpacks and of the
halo are computed once here (``SlabLayout``), so a CPU stand-in for the local kernels (the
world-size-2 gloo test) exercises exactly the layout and collective logic of the GPU path.

Buffers per rank (fp64): row slab [nt][nyl][n], column slab [nt][n][nxl], send / receive
buffers of the larger transpose block sum, halos [nt][2][n].
"""
from dataclasses import dataclass
from typing import List, Tuple

Desc = Tuple[Tuple[int, int, int], Tuple[int, int], Tuple[int, int], int, int]   # n, s, d, src_off, dst_off


def split(n: int, parts: int) -> List[Tuple[int, int]]:
    """Contiguous near-even split of range(n): (start, count) per part; the first n % parts parts
    get one extra element."""
    base, extra = divmod(n, parts)
    out, s = [], 0
    for p in range(parts):
        c = base + (1 if p < extra else 0)
        out.append((s, c))
        s += c
    return out


@dataclass
class SlabLayout:
    """Slab geometry of an n x n grid with nt slices over P ranks, and the copy descriptors
    (``paradiag_copy3d`` form) of every pack / unpack."""
    n: int
    nt: int
    P: int

    def __post_init__(self):
        self.rows = split(self.n, self.P)
        self.cols = split(self.n, self.P)
        if min(c for _, c in self.rows) < 3:
            raise ValueError("slab mode needs at least 3 rows per rank")

    # sizes (elements)
    def row_slab(self, r):
        return self.nt * self.rows[r][1] * self.n

    def col_slab(self, r):
        return self.nt * self.n * self.cols[r][1]

    def block(self, rr, cq):
        """elements of the (row slab rr) x (column slab cq) block of all slices"""
        return self.nt * self.rows[rr][1] * self.cols[cq][1]

    # forward transpose: rows -> columns
    def fwd_send_splits(self, r):
        return [self.block(r, q) for q in range(self.P)]

    def fwd_recv_splits(self, q):
        return [self.block(s, q) for s in range(self.P)]

    def fwd_pack(self, r) -> List[Desc]:
        """rows[r] slab [nt][nyl][n] -> send buffer, block q = [nt][nyl][nxl_q]"""
        nyl, out, off = self.rows[r][1], [], 0
        for q in range(self.P):
            x0, nxl = self.cols[q]
            out.append(((self.nt, nyl, nxl), (nyl * self.n, self.n), (nyl * nxl, nxl), x0, off))
            off += self.block(r, q)
        return out

    def fwd_unpack(self, q) -> List[Desc]:
        """receive buffer (block s = [nt][nyl_s][nxl]) -> column slab [nt][n][nxl] rows y_s.."""
        nxl, out, off = self.cols[q][1], [], 0
        for s in range(self.P):
            y0, nyl = self.rows[s]
            out.append(((self.nt, nyl, nxl), (nyl * nxl, nxl), (self.n * nxl, nxl), off, y0 * nxl))
            off += self.block(s, q)
        return out

    # backward transpose: columns -> rows (the mirror of the forward one)
    def bwd_send_splits(self, q):
        return self.fwd_recv_splits(q)

    def bwd_recv_splits(self, r):
        return self.fwd_send_splits(r)

    def bwd_pack(self, q) -> List[Desc]:
        return [(n, d, s, do, so) for (n, s, d, so, do) in self.fwd_unpack(q)]

    def bwd_unpack(self, r) -> List[Desc]:
        return [(n, d, s, do, so) for (n, s, d, so, do) in self.fwd_pack(r)]

    # transpose-block maps (paradiag_slab_*_seg): the passes next to a transpose address the
    # all-to-all buffers directly, so the packs / unpacks above are not copies at run time
    def xmap(self, r):
        """x-pass blocks of rank r: the forward send / backward receive buffer, block q =
        [nt][nyl_r][nxl_q] holding x ∈ cols[q]: [(x0_q, nxl_q, offset_q)]"""
        out, off = [], 0
        for q in range(self.P):
            x0, nxl = self.cols[q]
            out.append((x0, nxl, off))
            off += self.block(r, q)
        return out

    def ymap(self, q):
        """y-pass blocks of rank q: the forward receive / backward send buffer, block s =
        [nt][nyl_s][nxl_q] holding y ∈ rows[s]: [(y0_s, nyl_s, offset_s)]"""
        out, off = [], 0
        for s in range(self.P):
            y0, nyl = self.rows[s]
            out.append((y0, nyl, off))
            off += self.block(s, q)
        return out

    # residual halo: first / last two local rows of every slice, packed [nt][2][n]
    def halo_pack(self, r) -> Tuple[Desc, Desc]:
        nyl = self.rows[r][1]
        lo = ((self.nt, 2, self.n), (nyl * self.n, self.n), (2 * self.n, self.n), 0, 0)
        hi = ((self.nt, 2, self.n), (nyl * self.n, self.n), (2 * self.n, self.n), (nyl - 2) * self.n, 0)
        return lo, hi

    def halo_size(self):
        return self.nt * 2 * self.n


class GpuOps:
    """The local steps of one rank, in the sm_100a library (slab entry points)."""

    def __init__(self, problem, device, stream, y0, nyl, x0, nxl):
        from . import paradiag_init_slab, make_problem, pd_problem
        import torch
        self.problem = problem if isinstance(problem, pd_problem) else make_problem(problem)
        self.device = device
        self.torch = torch
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        self.h = paradiag_init_slab(self.problem, device, stream, y0, nyl, x0, nxl)

    def empty(self, count):
        return self.torch.empty(count, dtype=self.torch.float64, device=f"cuda:{self.device}")

    def copy(self, src, dst, desc: Desc):
        from . import paradiag_copy3d
        n, s, d, so, do = desc
        paradiag_copy3d(self.h, src, dst, n, s, d, so, do)

    def residual(self, u0_l, U_l, hlo, hhi, r_l):
        from . import paradiag_slab_residual
        paradiag_slab_residual(self.h, u0_l, U_l, hlo, hhi, r_l)

    def xpass(self, src, dst, want_dmax=False):
        from . import paradiag_slab_xpass
        paradiag_slab_xpass(self.h, src, dst, want_dmax)

    def ypass(self, cols):
        from . import paradiag_slab_ypass
        paradiag_slab_ypass(self.h, cols)

    def xrange(self, src, dst, want_dmax, seg_in, seg_out, n0, nn):
        from . import paradiag_slab_xrange
        paradiag_slab_xrange(self.h, src, dst, want_dmax, seg_in, seg_out, n0, nn)

    def yrange(self, src, cols, dst, stage, seg, n0, nn):
        from . import paradiag_slab_yrange
        paradiag_slab_yrange(self.h, src, cols, dst, stage, seg, n0, nn)

    def update_range(self, U_l, delta_l, n0, nn):
        from . import paradiag_slab_update_range
        paradiag_slab_update_range(self.h, U_l, delta_l, n0, nn)

    def xpass_seg(self, src, dst, want_dmax=False, seg_in=None, seg_out=None):
        from . import paradiag_slab_xpass_seg
        paradiag_slab_xpass_seg(self.h, src, dst, want_dmax, seg_in, seg_out)

    def ypass_seg(self, src, cols, dst, seg_in=None, seg_out=None):
        from . import paradiag_slab_ypass_seg
        paradiag_slab_ypass_seg(self.h, src, cols, dst, seg_in, seg_out)

    def update(self, U_l, delta_l):
        from . import paradiag_slab_update
        paradiag_slab_update(self.h, U_l, delta_l)

    def stats_reset(self):
        from . import paradiag_stats_reset
        paradiag_stats_reset(self.h)

    def stats_read(self):
        from . import paradiag_stats_read
        return paradiag_stats_read(self.h)

    def close(self):
        from . import paradiag_destroy
        if self.h:
            paradiag_destroy(self.h)
            self.h = None


class TorchComm:
    """Collectives of a real multi-process run (torch.distributed, NCCL or gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_to_all(self, recv, send, recv_splits, send_splits, async_op=False):
        """async_op: return the work handle; wait() on it orders the caller's stream after the
        collective (NCCL) or blocks until it is done (gloo)."""
        return self.dist.all_to_all_single(recv[:sum(recv_splits)], send[:sum(send_splits)], recv_splits,
                                           send_splits, group=self.group, async_op=async_op)

    def halo(self, send_lo, send_hi, recv_lo, recv_hi):
        """send_lo -> rank-1 (its upper halo), send_hi -> rank+1 (its lower halo)"""
        ops = []
        P2P = self.dist.P2POp
        if self.rank > 0:
            ops += [P2P(self.dist.isend, send_lo, self.rank - 1, self.group),
                    P2P(self.dist.irecv, recv_lo, self.rank - 1, self.group)]
        if self.rank < self.world - 1:
            ops += [P2P(self.dist.isend, send_hi, self.rank + 1, self.group),
                    P2P(self.dist.irecv, recv_hi, self.rank + 1, self.group)]
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def shift_up(self, send, recv):
        """One-directional neighbour exchange: send -> rank+1, recv <- rank-1 (separate buffers, no
        message in the unused direction)."""
        ops = []
        P2P = self.dist.P2POp
        if self.rank < self.world - 1:
            ops.append(P2P(self.dist.isend, send, self.rank + 1, self.group))
        if self.rank > 0:
            ops.append(P2P(self.dist.irecv, recv, self.rank - 1, self.group))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def allreduce_max(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)

    def fence(self):
        """Stream-ordered barrier (a one-element NCCL all-reduce): every rank's preceding kernels,
        including their peer-memory stores, complete before anyone's following kernels start."""
        if not hasattr(self, "_tok"):
            import torch
            self._tok = torch.zeros(1, dtype=torch.float64, device=torch.cuda.current_device())
        self.dist.all_reduce(self._tok, group=self.group)

    def all_gather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


class SlabRank:
    """State and phases of one rank.  ``iterate`` runs one defect-correction iteration
    U ← U + P_α⁻¹(b − K U) on the rank's row slab."""

    def __init__(self, layout: SlabLayout, rank: int, ops, fused: bool = True, chunks: int = 1, p2p: bool = False,
                 self_via_comm: bool = False):
        """fused: the x / y passes read and write the all-to-all buffers through the block maps
        (no pack / unpack copies); False: the copy-based reference orchestration.
        chunks > 1 (fused only): the time slices are cut into that many ranges, each with its own
        blocks in the buffer, so the all-to-all of one range runs (async) while the passes work on
        the next (the time pass in the middle needs every slice and waits for all of them)."""
        self.L, self.r, self.ops = layout, rank, ops
        self.fused = fused or p2p
        self.p2p = p2p
        self.peer = None                                   # p2p: peer buffer addresses (connect_p2p)
        self.chunks = 1 if p2p else (max(1, min(chunks, layout.nt)) if fused else 1)
        self.ranges = split(layout.nt, self.chunks)
        self.y0, self.nyl = layout.rows[rank]
        self.x0, self.nxl = layout.cols[rank]
        P, r = layout.P, rank
        self.rows = ops.empty(layout.row_slab(rank))         # r, then δ
        self.cols = ops.empty(layout.col_slab(rank))
        if p2p:
            # peer-memory transposes: [recv_f | recv_b | self]; the x pass and the inverse y pass
            # store their peer blocks straight into the peers' receive regions (maps set by
            # connect_p2p once the peers' addresses are known), NCCL only fences
            fs = [0 if q == r else layout.block(r, q) for q in range(P)]
            fr = [0 if q == r else layout.block(q, r) for q in range(P)]
            self.p2p_sizes = (sum(fr), sum(fs))
            self.buf = ops.empty(sum(fr) + sum(fs) + layout.block(r, r))
            self.send = self.recv = None
            self.splits = {"fwd": ([0] * P, [0] * P), "bwd": ([0] * P, [0] * P)}
        elif self.fused:
            # per slice range one region [send | recv | self] of a single buffer: the block a rank
            # keeps (row slab r ∩ column slab r) goes straight from the x pass to the y pass through
            # the self region and is left out of the collective (split 0), so NCCL moves only the
            # peer blocks.  Blocks of a range are [nn][rows][cols] (range-relative addressing).
            cum = lambda sp: [sum(sp[:i]) for i in range(P)]
            regions, base = [], 0
            # self_via_comm (test hook): the kept block also travels through the collective, so a
            # one-rank NCCL run exercises the asynchronous all-to-all and its stream ordering
            keep = not self_via_comm
            for n0, nn in self.ranges:
                fs = [0 if (q == r and keep) else nn * self.nyl * layout.cols[q][1] for q in range(P)]   # fwd send / bwd recv
                fr = [0 if (q == r and keep) else nn * layout.rows[q][1] * self.nxl for q in range(P)]  # fwd recv / bwd send
                ns = max(sum(fs), sum(fr))
                so = base + 2 * ns                                              # the self block
                cfs, cfr = cum(fs), cum(fr)
                own = lambda q: q == r and keep
                regions.append(dict(
                    n0=n0, nn=nn, base=base, ns=ns, splits={"fwd": (fs, fr), "bwd": (fr, fs)},
                    xm_out=[(x0, c, so if own(q) else base + cfs[q]) for q, (x0, c) in enumerate(layout.cols)],
                    ym_in=[(y0, c, so if own(q) else base + ns + cfr[q]) for q, (y0, c) in enumerate(layout.rows)],
                    ym_out=[(y0, c, so if own(q) else base + cfr[q]) for q, (y0, c) in enumerate(layout.rows)],
                    xm_in=[(x0, c, so if own(q) else base + ns + cfs[q]) for q, (x0, c) in enumerate(layout.cols)]))
                base = so + (nn * self.nyl * self.nxl if keep else 0)
            self.buf = ops.empty(base)
            for g in regions:
                g["send"] = self.buf[g["base"]:g["base"] + g["ns"]]
                g["recv"] = self.buf[g["base"] + g["ns"]:g["base"] + 2 * g["ns"]]
            self.regions = regions
            # whole-range aliases (chunks = 1)
            g = regions[0]
            self.splits, self.send, self.recv = g["splits"], g["send"], g["recv"]
            self.xm_out, self.ym_in, self.ym_out, self.xm_in = g["xm_out"], g["ym_in"], g["ym_out"], g["xm_in"]
        else:
            self.splits = {"fwd": (layout.fwd_send_splits(r), layout.fwd_recv_splits(r)),
                           "bwd": (layout.bwd_send_splits(r), layout.bwd_recv_splits(r))}
            tsz = max(sum(layout.fwd_send_splits(rank)), sum(layout.fwd_recv_splits(rank)))
            self.send = ops.empty(tsz)
            self.recv = ops.empty(tsz)
        hs = layout.halo_size()
        self.hsend_lo, self.hsend_hi = ops.empty(hs), ops.empty(hs)
        self.hlo = ops.empty(hs) if rank > 0 else None
        self.hhi = ops.empty(hs) if rank < P - 1 else None
        self._dummy = ops.empty(hs) if (self.hlo is None or self.hhi is None) else None

    # ---- phases (each only enqueues local work)
    def phase_halo_pack(self, U_l):
        lo, hi = self.L.halo_pack(self.r)
        self.ops.stats_reset()
        self.ops.copy(U_l, self.hsend_lo, lo)
        self.ops.copy(U_l, self.hsend_hi, hi)

    def phase_residual_xfwd(self, u0_l, U_l):
        self.ops.residual(u0_l, U_l, self.hlo, self.hhi, self.rows)
        if self.fused:                                   # x pass stores straight into the send blocks
            self.ops.xpass_seg(self.rows, self.buf, False, None, self.xm_out)
            return
        self.ops.xpass(self.rows, self.rows)
        for d in self.L.fwd_pack(self.r):
            self.ops.copy(self.rows, self.send, d)

    def phase_ypass(self):
        if self.fused:                                   # receive blocks -> cols -> send blocks
            self.ops.ypass_seg(self.buf, self.cols, self.buf, self.ym_in, self.ym_out)
            return
        for d in self.L.fwd_unpack(self.r):
            self.ops.copy(self.recv, self.cols, d)
        self.ops.ypass(self.cols)
        for d in self.L.bwd_pack(self.r):
            self.ops.copy(self.cols, self.send, d)

    def phase_xinv_update(self, U_l):
        if self.fused:                                   # inverse x pass loads the receive blocks
            self.ops.xpass_seg(self.buf, self.rows, True, self.xm_in, None)
        else:
            for d in self.L.bwd_unpack(self.r):
                self.ops.copy(self.recv, self.rows, d)
            self.ops.xpass(self.rows, self.rows, want_dmax=True)
        self.ops.update(U_l, self.rows)

    def _alltoall(self, comm, tm, phase):
        if self.p2p:                                     # the blocks were stored into the peers: fence
            with tm("p2p_fence_" + phase):
                comm.fence()
            return
        ssp, rsp = self.splits[phase]
        if sum(ssp) + sum(rsp) == 0:                     # P = 1 with the fused layout: nothing to move
            return
        with tm("alltoall_" + phase):
            comm.all_to_all(self.recv, self.send, rsp, ssp)

    # ---- peer-memory transposes
    def p2p_layout(self, q):
        """(recv_f base, recv_b base, fwd-recv block offsets, bwd-recv block offsets) of rank q's
        buffer, in elements"""
        L, P = self.L, self.L.P
        fr_q = [0 if s == q else L.block(s, q) for s in range(P)]
        fs_q = [0 if t == q else L.block(q, t) for t in range(P)]
        cum = lambda sp: [sum(sp[:i]) for i in range(P)]
        return 0, sum(fr_q), cum(fr_q), cum(fs_q)

    def connect_p2p(self, peer_addr):
        """peer_addr[q]: device address (in this process) of rank q's buffer; builds the maps whose
        peer blocks are element offsets from this rank's own buffer."""
        L, P, r = self.L, self.L.P, self.r
        self.peer = list(peer_addr)
        me = self.peer[r]
        rf, rb, cfr, cfs = self.p2p_layout(r)
        so = rb + sum(0 if t == r else L.block(r, t) for t in range(P))     # self region
        rel = lambda q: (self.peer[q] - me) // 8
        xm_out, ym_out = [], []
        for q, (x0, c) in enumerate(L.cols):
            if q == r:
                xm_out.append((x0, c, so))
            else:
                qf, _, qcfr, _ = self.p2p_layout(q)
                xm_out.append((x0, c, rel(q) + qf + qcfr[r]))      # my block in q's forward receive region
        for s_, (y0, c) in enumerate(L.rows):
            if s_ == r:
                ym_out.append((y0, c, so))
            else:
                _, sb, _, scfs = self.p2p_layout(s_)
                ym_out.append((y0, c, rel(s_) + sb + scfs[r]))     # my block in s's backward receive region
        self.xm_out, self.ym_out = xm_out, ym_out
        self.ym_in = [(y0, c, so if q == r else rf + cfr[q]) for q, (y0, c) in enumerate(L.rows)]
        self.xm_in = [(x0, c, so if q == r else rb + cfs[q]) for q, (x0, c) in enumerate(L.cols)]

    def setup_p2p(self, comm):
        """Real multi-process run: export this rank's buffer (CUDA IPC), map every peer's."""
        from . import paradiag_ipc_handle, paradiag_ipc_open
        import cuda.bindings.driver as drv
        ptr = self.buf.data_ptr()
        err, base, _ = drv.cuMemGetAddressRange(ptr)
        base = int(base)
        if err != drv.CUresult.CUDA_SUCCESS:
            raise RuntimeError(f"cuMemGetAddressRange: {err}")
        info = (paradiag_ipc_handle(base), ptr - base)     # handle of the allocation, tensor offset
        allinfo = comm.all_gather_object(info)
        peer = []
        self._mapped = []
        for q, (hd, off) in enumerate(allinfo):
            if q == self.r:
                peer.append(ptr)
            else:
                b = paradiag_ipc_open(hd)
                self._mapped.append(b)
                peer.append(b + off)
        self.connect_p2p(peer)

    def close_p2p(self):
        """Unmap the peers' buffers (setup_p2p)."""
        from . import paradiag_ipc_close
        for b in getattr(self, "_mapped", []):
            paradiag_ipc_close(b)
        self._mapped = []

    # ---- chunked phases (chunks > 1): range c's collective overlaps the passes of range c+1
    def chunk_xfwd(self, c):
        g = self.regions[c]
        self.ops.xrange(self.rows, self.buf, False, None, g["xm_out"], g["n0"], g["nn"])

    def chunk_yfwd(self, c):
        g = self.regions[c]
        self.ops.yrange(self.buf, self.cols, self.cols, 0, g["ym_in"], g["n0"], g["nn"])

    def phase_time(self):
        self.ops.yrange(self.cols, self.cols, self.cols, 1, None, 0, self.L.nt)

    def chunk_yinv(self, c):
        g = self.regions[c]
        self.ops.yrange(self.cols, self.cols, self.buf, 2, g["ym_out"], g["n0"], g["nn"])

    def chunk_xinv_update(self, c, U_l):
        g = self.regions[c]
        self.ops.xrange(self.buf, self.rows, True, g["xm_in"], None, g["n0"], g["nn"])
        self.ops.update_range(U_l, self.rows, g["n0"], g["nn"])

    def _alltoall_chunk(self, comm, c, phase):
        g = self.regions[c]
        ssp, rsp = g["splits"][phase]
        if sum(ssp) + sum(rsp) == 0:
            return None
        return comm.all_to_all(g["recv"], g["send"], rsp, ssp, async_op=True)

    def _iterate_chunked(self, u0_l, U_l, comm, tm):
        self.ops.residual(u0_l, U_l, self.hlo, self.hhi, self.rows)
        C = len(self.regions)
        works = []
        for c in range(C):                                # x pass of range c, then its transpose in flight
            self.chunk_xfwd(c)
            works.append(self._alltoall_chunk(comm, c, "fwd"))
        with tm("alltoall_fwd_tail"):
            for c in range(C):
                if works[c] is not None:
                    works[c].wait()
                self.chunk_yfwd(c)
        self.phase_time()
        works = []
        for c in range(C):
            self.chunk_yinv(c)
            works.append(self._alltoall_chunk(comm, c, "bwd"))
        with tm("alltoall_bwd_tail"):
            for c in range(C):
                if works[c] is not None:
                    works[c].wait()
                self.chunk_xinv_update(c, U_l)

    # ---- one iteration of a real multi-process run
    def iterate(self, u0_l, U_l, comm: TorchComm, timer=None):
        """timer: optional callable(name) -> context manager timing a collective on the device"""
        L, r = self.L, self.r
        tm = timer or (lambda name: _Null())
        self.phase_halo_pack(U_l)
        with tm("halo"):
            comm.halo(self.hsend_lo, self.hsend_hi, self.hlo if self.hlo is not None else self._dummy,
                      self.hhi if self.hhi is not None else self._dummy)
        if self.chunks > 1:
            self._iterate_chunked(u0_l, U_l, comm, tm)
            dmax, umax = self.ops.stats_read()
            t = self.ops.empty(2)
            t[0], t[1] = dmax, umax
            comm.allreduce_max(t)
            return float(t[0]), float(t[1])
        self.phase_residual_xfwd(u0_l, U_l)
        self._alltoall(comm, tm, "fwd")
        self.phase_ypass()
        self._alltoall(comm, tm, "bwd")
        self.phase_xinv_update(U_l)
        dmax, umax = self.ops.stats_read()
        t = self.ops.empty(2) if hasattr(self.ops, "empty") else None
        t[0], t[1] = dmax, umax
        comm.allreduce_max(t)
        return float(t[0]), float(t[1])


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def iterate_virtual(ranks: List[SlabRank], u0s, Us):
    """All P ranks of a layout in ONE process (one GPU): the same phases in rank order with the
    collectives emulated by buffer copies — the multi-rank data path checked on a single device
    (no rank waits on another, so nothing can deadlock)."""
    P = len(ranks)
    L = ranks[0].L
    for k in range(P):
        ranks[k].phase_halo_pack(Us[k])
    for k in range(P):
        if k > 0:
            ranks[k].hlo.copy_(ranks[k - 1].hsend_hi)
        if k < P - 1:
            ranks[k].hhi.copy_(ranks[k + 1].hsend_lo)
    if ranks[0].chunks > 1:
        return _iterate_virtual_chunked(ranks, u0s, Us)
    if ranks[0].p2p and ranks[0].peer is None:           # one process: the peers' buffers are local
        addr = [rk.buf.data_ptr() for rk in ranks]
        for rk in ranks:
            rk.connect_p2p(addr)
    for k in range(P):
        ranks[k].phase_residual_xfwd(u0s[k], Us[k])
    _alltoall_virtual(ranks, "fwd")
    for k in range(P):
        ranks[k].phase_ypass()
    _alltoall_virtual(ranks, "bwd")
    for k in range(P):
        ranks[k].phase_xinv_update(Us[k])
    st = [rk.ops.stats_read() for rk in ranks]
    return max(s[0] for s in st), max(s[1] for s in st)


def _iterate_virtual_chunked(ranks, u0s, Us):
    """The chunked schedule with the per-range transposes emulated by copies."""
    P = len(ranks)
    C = len(ranks[0].regions)
    for k in range(P):
        ranks[k].ops.residual(u0s[k], Us[k], ranks[k].hlo, ranks[k].hhi, ranks[k].rows)
    for c in range(C):
        for k in range(P):
            ranks[k].chunk_xfwd(c)
        _alltoall_virtual(ranks, "fwd", c)
        for k in range(P):
            ranks[k].chunk_yfwd(c)
    for k in range(P):
        ranks[k].phase_time()
    for c in range(C):
        for k in range(P):
            ranks[k].chunk_yinv(c)
        _alltoall_virtual(ranks, "bwd", c)
        for k in range(P):
            ranks[k].chunk_xinv_update(c, Us[k])
    st = [rk.ops.stats_read() for rk in ranks]
    return max(s[0] for s in st), max(s[1] for s in st)


def _alltoall_virtual(ranks, phase, chunk=None):
    P = len(ranks)
    if ranks[0].p2p:                                     # stored directly into the peers' regions
        return
    if chunk is not None:
        send_splits = [rk.regions[chunk]["splits"][phase][0] for rk in ranks]
        sends = [rk.regions[chunk]["send"] for rk in ranks]
        recvs = [rk.regions[chunk]["recv"] for rk in ranks]
    else:
        send_splits = [rk.splits[phase][0] for rk in ranks]
        sends = [rk.send for rk in ranks]
        recvs = [rk.recv for rk in ranks]
    soff = [[sum(send_splits[s][:q]) for q in range(P)] for s in range(P)]
    for q in range(P):
        off = 0
        for s in range(P):
            c = send_splits[s][q]
            recvs[q][off:off + c].copy_(sends[s][soff[s][q]:soff[s][q] + c])
            off += c


# ---------------------------------------------------------------------------------------------
# Time slabs: 1D long windows across ranks ("frequency sharding with a tiny
# spatial problem — the other aspect ratio").  With N_x ≤ 64 and N_t up to 2^20 the
# natural cut is in time: rank r owns the time rows [r·nn, (r+1)·nn) of U (nn = N_t / P) for the
# residual (row n couples only u_n and u_{n-1}, so the one halo row is the previous
# rank's last row, u0 on rank 0), the x transforms (DST-I / DCT-I per row) and the update; for
# Steps (1)-(3) (per spatial mode along the whole window) it owns the x-mode block
# [r·bc, (r+1)·bc) of every time row (bc = pitch / P, pitch = 2⌈N_x/2⌉).  Per iteration:
#   halo row → residual + x transform into [P][nn][bc] blocks → all-to-all (block q to rank q;
#   the received blocks stack to [N_t][bc]) → four-step time pass with the per-bin divide on the
#   local modes → all-to-all back → inverse x transform + update → max-reduce ‖δ‖∞, ‖U‖∞.
# Every step is a library call (paradiag_tslab_* of include/paradiag.h) through ``TslabOps``.
class TslabOps:
    """The local steps of one time-slab rank: a handle of the GLOBAL problem on this device."""

    def __init__(self, problem, device, stream=None):
        from . import paradiag_init, make_problem, pd_problem, paradiag_tslab_pitch
        import torch
        self.problem = problem if isinstance(problem, pd_problem) else make_problem(problem)
        self.device = device
        self.torch = torch
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        self.h = paradiag_init(self.problem, device, stream)
        self.pitch = paradiag_tslab_pitch(self.h)
        self.nt = int(self.problem.nt)
        self.nx = int(self.problem.m) + (1 if int(self.problem.bc) == 0 else -1)

    def empty(self, count):
        return self.torch.empty(count, dtype=self.torch.float64, device=f"cuda:{self.device}")

    def residual(self, u_prev, U_l, nn, blocks, bc):
        from . import paradiag_tslab_residual
        paradiag_tslab_residual(self.h, u_prev, U_l, nn, blocks, bc)

    def time(self, cols, c0, bc):
        from . import paradiag_tslab_time
        paradiag_tslab_time(self.h, cols, c0, bc)

    def update(self, blocks, bc, U_l, nn):
        from . import paradiag_tslab_update
        paradiag_tslab_update(self.h, blocks, bc, U_l, nn)

    def stats_reset(self):
        from . import paradiag_stats_reset
        paradiag_stats_reset(self.h)

    def stats_read(self):
        from . import paradiag_stats_read
        return paradiag_stats_read(self.h)

    def close(self):
        from . import paradiag_destroy
        if self.h:
            paradiag_destroy(self.h)
            self.h = None


def tslab_geometry(nt: int, pitch: int, world: int):
    """(nn, bc): time rows per rank and x-modes per rank; P must divide N_t and pitch/2."""
    if world < 1 or nt % world or pitch % world or (pitch // world) % 2:
        raise ValueError(f"time slabs: {world} ranks must divide N_t = {nt} and pitch/2 = {pitch // 2}")
    return nt // world, pitch // world


class TimeSlabRank:
    """State and phases of one time-slab rank; ``iterate`` runs one defect-correction iteration on
    the rank's rows U_l [nn][N_x] (flat)."""

    def __init__(self, ops, rank: int, world: int):
        self.ops, self.r, self.P = ops, rank, world
        self.nt, self.nx, self.pitch = ops.nt, ops.nx, ops.pitch
        self.nn, self.bc = tslab_geometry(self.nt, self.pitch, world)
        self.n0, self.c0 = rank * self.nn, rank * self.bc
        self.blocks = ops.empty(world * self.nn * self.bc)     # [P][nn][bc]: residual out / update in
        self.cols = ops.empty(self.nt * self.bc)               # [N_t][bc] = [P][nn][bc]
        self.halo = ops.empty(self.nx)                         # u_{n0-1} from rank r-1
        self.splits = [self.nn * self.bc] * world

    def last_row(self, U_l):
        return U_l[(self.nn - 1) * self.nx:self.nn * self.nx]

    def phase_residual(self, u0, U_l):
        self.ops.stats_reset()
        self.ops.residual(u0 if self.r == 0 else self.halo, U_l, self.nn, self.blocks, self.bc)

    def phase_time(self):
        self.ops.time(self.cols, self.c0, self.bc)

    def phase_update(self, U_l):
        self.ops.update(self.blocks, self.bc, U_l, self.nn)

    def iterate(self, u0, U_l, comm: TorchComm, timer=None):
        tm = timer or (lambda name: _Null())
        with tm("halo"):      # last row → rank r+1 (its u_{n0-1}), one direction only
            comm.shift_up(self.last_row(U_l).contiguous(), self.halo)
        self.phase_residual(u0, U_l)
        with tm("all_to_all"):
            comm.all_to_all(self.cols, self.blocks, self.splits, self.splits)
        self.phase_time()
        with tm("all_to_all"):
            comm.all_to_all(self.blocks, self.cols, self.splits, self.splits)
        self.phase_update(U_l)
        dmax, umax = self.ops.stats_read()
        t = self.ops.empty(2)
        t[0], t[1] = dmax, umax
        comm.allreduce_max(t)
        return float(t[0]), float(t[1])


def iterate_tslab_virtual(ranks: List[TimeSlabRank], u0, Us):
    """All P time-slab ranks in ONE process (one GPU): the phases in rank order, the halo and the
    all-to-alls emulated by copies (no rank waits on another)."""
    P = len(ranks)
    for k in range(1, P):
        ranks[k].halo.copy_(ranks[k - 1].last_row(Us[k - 1]))
    for k in range(P):
        ranks[k].phase_residual(u0, Us[k])
    _tslab_exchange([rk.blocks for rk in ranks], [rk.cols for rk in ranks], ranks[0].splits[0])
    for k in range(P):
        ranks[k].phase_time()
    _tslab_exchange([rk.cols for rk in ranks], [rk.blocks for rk in ranks], ranks[0].splits[0])
    for k in range(P):
        ranks[k].phase_update(Us[k])
    st = [rk.ops.stats_read() for rk in ranks]
    return max(s[0] for s in st), max(s[1] for s in st)


def _tslab_exchange(sends, recvs, c):
    """all_to_all with equal chunks c: chunk q of rank s's send → chunk s of rank q's receive."""
    P = len(sends)
    for q in range(P):
        for s in range(P):
            recvs[q][s * c:(s + 1) * c].copy_(sends[s][q * c:(q + 1) * c])
