"""Multi-rank orchestration on CPU: world size 2 over torch.distributed gloo.

paper_2304_14021_b200/dist.py (slab layout, copy descriptors, halo exchange, all-to-all splits,
reductions) runs with real gloo collectives; the local kernels are replaced by a CPU stand-in built
from the oracle's transforms (this file), so the test checks the multi-rank data movement against
the oracle's unsharded iteration.  The same layout code drives the GPU path (tests/test_gpu_dist.py
runs it with the real kernels as virtual ranks on one device)."""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import circulant, iterate, spatial, precond
from workloads import twin, make_u0

CASES = {"neumann": twin("c5", m=32, nt=8), "hinged": twin("c3", m=32, nt=8)}


class CpuOps:
    """CPU stand-in for dist.GpuOps (same conventions: unnormalised x/y transforms, the time pass
    carries Γ_α, the per-mode divide, 1/N_t and the spatial 1/(2m)²)."""

    def __init__(self, p, y0, nyl, x0, nxl):
        self.p, self.y0, self.nyl, self.x0, self.nxl = p, y0, nyl, x0, nxl
        self.n = p.n
        self.T = spatial.transform_matrix(p.m, p.bc)
        self.dmax = self.umax = 0.0

    def empty(self, count):
        return torch.zeros(count, dtype=torch.float64)

    def copy(self, src, dst, desc):
        (n0, n1, n2), (s0, s1), (d0, d1), so, do = desc
        sv = src.as_strided((n0, n1, n2), (s0, s1, 1), src.storage_offset() + so)
        dv = dst.as_strided((n0, n1, n2), (d0, d1, 1), dst.storage_offset() + do)
        dv.copy_(sv)

    def residual(self, u0_l, U_l, hlo, hhi, r_l):
        p, n, nt = self.p, self.n, self.p.nt
        full = np.zeros((nt, n, n))
        full[:, self.y0:self.y0 + self.nyl] = U_l.numpy().reshape(nt, self.nyl, n)
        if hlo is not None:
            full[:, self.y0 - 2:self.y0] = hlo.numpy().reshape(nt, 2, n)
        if hhi is not None:
            full[:, self.y0 + self.nyl:self.y0 + self.nyl + 2] = hhi.numpy().reshape(nt, 2, n)
        u0 = np.zeros((n, n))
        u0[self.y0:self.y0 + self.nyl] = u0_l.numpy().reshape(self.nyl, n)
        r, _ = iterate.residual(p, u0, full)        # nested 5-point stencil: rows ±2 suffice
        r_l.copy_(torch.from_numpy(np.ascontiguousarray(r[:, self.y0:self.y0 + self.nyl]).reshape(-1)))

    def xpass(self, src, dst, want_dmax=False):
        a = src.numpy().reshape(self.p.nt, self.nyl, self.n) @ self.T.T
        if want_dmax:
            self.dmax = max(self.dmax, float(np.abs(a).max()))
        dst.copy_(torch.from_numpy(np.ascontiguousarray(a).reshape(-1)))

    def ypass(self, cols):
        p, nt, n = self.p, self.p.nt, self.n
        c = cols.numpy().reshape(nt, n, self.nxl)
        hat = np.einsum("qy,tyx->tqx", self.T, c)
        S = circulant.step1(hat, p.alpha)
        d = circulant.eig_d(nt, p.alpha, circulant.inv_dt(p))
        mu = precond._step2_mu(p, 0.0)[:, self.x0:self.x0 + self.nxl]          # [q, p_local]
        S = S / (d[:, None, None] + mu[None])
        x, _ = circulant.step3(S, p.alpha)
        out = np.einsum("qy,tyx->tqx", self.T, x) / (2.0 * p.m) ** 2
        cols.copy_(torch.from_numpy(np.ascontiguousarray(out).reshape(-1)))

    # transpose-block variants (the maps of SlabLayout.xmap / ymap): gather, run, scatter
    def _gather_x(self, src, seg):
        nt, nyl, n = self.p.nt, self.nyl, self.n
        if seg is None:
            return src.numpy().reshape(nt, nyl, n)
        out = np.empty((nt, nyl, n))
        for x0, cnt, off in seg:
            out[:, :, x0:x0 + cnt] = src.numpy()[off:off + nt * nyl * cnt].reshape(nt, nyl, cnt)
        return out

    def _scatter_x(self, a, dst, seg):
        nt, nyl = self.p.nt, self.nyl
        if seg is None:
            dst.copy_(torch.from_numpy(np.ascontiguousarray(a).reshape(-1)))
            return
        for x0, cnt, off in seg:
            dst[off:off + nt * nyl * cnt] = torch.from_numpy(np.ascontiguousarray(a[:, :, x0:x0 + cnt]).reshape(-1))

    def xpass_seg(self, src, dst, want_dmax=False, seg_in=None, seg_out=None):
        a = self._gather_x(src, seg_in) @ self.T.T
        if want_dmax:
            self.dmax = max(self.dmax, float(np.abs(a).max()))
        self._scatter_x(a, dst, seg_out)

    def ypass_seg(self, src, cols, dst, seg_in=None, seg_out=None):
        nt, n, nxl = self.p.nt, self.n, self.nxl
        if seg_in is None:
            cols.copy_(src)
        else:
            c = np.empty((nt, n, nxl))
            for y0, cnt, off in seg_in:
                c[:, y0:y0 + cnt, :] = src.numpy()[off:off + nt * cnt * nxl].reshape(nt, cnt, nxl)
            cols.copy_(torch.from_numpy(c.reshape(-1)))
        self.ypass(cols)
        if seg_out is None:
            dst.copy_(cols)
            return
        c = cols.numpy().reshape(nt, n, nxl)
        for y0, cnt, off in seg_out:
            dst[off:off + nt * cnt * nxl] = torch.from_numpy(np.ascontiguousarray(c[:, y0:y0 + cnt, :]).reshape(-1))

    # slice-range forms (chunked schedule): slab buffers from slice 0, blocks range-relative
    def xrange(self, src, dst, want_dmax, seg_in, seg_out, n0, nn):
        nyl, n = self.nyl, self.n
        if seg_in is None:
            a = src.numpy().reshape(self.p.nt, nyl, n)[n0:n0 + nn]
        else:
            a = np.empty((nn, nyl, n))
            for x0, cnt, off in seg_in:
                a[:, :, x0:x0 + cnt] = src.numpy()[off:off + nn * nyl * cnt].reshape(nn, nyl, cnt)
        a = a @ self.T.T
        if want_dmax:
            self.dmax = max(self.dmax, float(np.abs(a).max()))
        if seg_out is None:
            dst.view(self.p.nt, nyl, n)[n0:n0 + nn] = torch.from_numpy(np.ascontiguousarray(a))
        else:
            for x0, cnt, off in seg_out:
                dst[off:off + nn * nyl * cnt] = torch.from_numpy(np.ascontiguousarray(a[:, :, x0:x0 + cnt]).reshape(-1))

    def yrange(self, src, cols, dst, stage, seg, n0, nn):
        p, nt, n, nxl = self.p, self.p.nt, self.n, self.nxl
        cv = cols.view(nt, n, nxl)
        if stage == 0:
            c = np.empty((nn, n, nxl))
            for y0, cnt, off in seg:
                c[:, y0:y0 + cnt, :] = src.numpy()[off:off + nn * cnt * nxl].reshape(nn, cnt, nxl)
            cv[n0:n0 + nn] = torch.from_numpy(np.einsum("qy,tyx->tqx", self.T, c))
        elif stage == 1:
            S = circulant.step1(cv.numpy(), p.alpha)
            d = circulant.eig_d(nt, p.alpha, circulant.inv_dt(p))
            mu = precond._step2_mu(p, 0.0)[:, self.x0:self.x0 + nxl]
            x, _ = circulant.step3(S / (d[:, None, None] + mu[None]), p.alpha)
            cv.copy_(torch.from_numpy(np.ascontiguousarray(x)))
        else:
            out = np.einsum("qy,tyx->tqx", self.T, cv.numpy()[n0:n0 + nn]) / (2.0 * p.m) ** 2
            for y0, cnt, off in seg:
                dst[off:off + nn * cnt * nxl] = torch.from_numpy(np.ascontiguousarray(out[:, y0:y0 + cnt, :]).reshape(-1))

    def update_range(self, U_l, delta_l, n0, nn):
        sl = slice(n0 * self.nyl * self.n, (n0 + nn) * self.nyl * self.n)
        U_l[sl] += delta_l[sl]
        self.umax = max(self.umax, float(U_l[sl].abs().max()))

    def update(self, U_l, delta_l):
        U_l += delta_l
        self.umax = max(self.umax, float(U_l.abs().max()))

    def stats_reset(self):
        self.dmax = self.umax = 0.0

    def stats_read(self):
        return self.dmax, self.umax


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, K, out, fused=True, chunks=1):
    import torch.distributed as dist
    from paper_2304_14021_b200 import dist as pdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = CASES[name]
        u0 = make_u0(p)
        U0 = iterate.initial_iterate(p, u0)
        L = pdist.SlabLayout(p.n, p.nt, world)
        y0, nyl = L.rows[rank]
        x0, nxl = L.cols[rank]
        ops = CpuOps(p, y0, nyl, x0, nxl)
        rk = pdist.SlabRank(L, rank, ops, fused=fused, chunks=chunks)
        comm = pdist.TorchComm()
        U_l = torch.from_numpy(np.ascontiguousarray(U0[:, y0:y0 + nyl]).reshape(-1))
        u0_l = torch.from_numpy(np.ascontiguousarray(u0[y0:y0 + nyl]))
        stats = []
        for _ in range(K):
            stats.append(rk.iterate(u0_l, U_l, comm))
        gathered = [torch.zeros(L.row_slab(r), dtype=torch.float64) for r in range(world)]
        dist.all_gather(gathered, U_l) if len(set(L.row_slab(r) for r in range(world))) == 1 else \
            [dist.broadcast(g.copy_(U_l) if r == rank else g, src=r) for r, g in enumerate(gathered)]
        if rank == 0:
            full = np.concatenate([g.numpy().reshape(p.nt, L.rows[r][1], p.n) for r, g in enumerate(gathered)], axis=1)
            np.save(out, full)
            np.save(out + ".stats.npy", np.array(stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", [(True, 1), (False, 1), (True, 3)], ids=["block-io", "pack-copies", "chunked3"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_two_rank_gloo_iteration_matches_oracle(tmp_path, name, mode):
    import torch.multiprocessing as mp
    p = CASES[name]
    K = 2
    out = str(tmp_path / "U.npy")
    mp.spawn(_worker, args=(2, _free_port(), name, K, out, mode[0], mode[1]), nprocs=2, join=True)
    got = np.load(out)
    stats = np.load(out + ".stats.npy")
    u0 = make_u0(p)
    U = iterate.initial_iterate(p, u0)
    for k in range(K):
        U, info = iterate.iterate_once(p, u0, U)
        # ‖δ‖∞ to rounding at the scale of the iterate (late increments are small against ‖U‖)
        assert abs(stats[k][0] - info["delta_max"]) <= 1e-11 * max(info["u_max"], info["delta_max"])
        assert abs(stats[k][1] - info["u_max"]) <= 1e-11 * info["u_max"]
    assert np.abs(got - U).max() <= 1e-11 * np.abs(U).max()


def test_layout_descriptors_cover_every_element():
    from paper_2304_14021_b200.dist import SlabLayout
    for n, nt, P in [(33, 4, 2), (33, 4, 3), (127, 2, 8), (2049, 1, 8)]:
        L = SlabLayout(n, nt, P)
        assert sum(c for _, c in L.rows) == n and sum(c for _, c in L.cols) == n
        for r in range(P):
            # forward pack reads every row-slab element exactly once
            seen = np.zeros(L.row_slab(r), dtype=np.int64)
            for (n0, n1, n2), (s0, s1), (d0, d1), so, do in L.fwd_pack(r):
                idx = so + np.arange(n0)[:, None, None] * s0 + np.arange(n1)[None, :, None] * s1 + np.arange(n2)
                np.add.at(seen, idx.reshape(-1), 1)
            assert (seen == 1).all()
            # forward unpack writes every column-slab element exactly once
            seen = np.zeros(L.col_slab(r), dtype=np.int64)
            for (n0, n1, n2), (s0, s1), (d0, d1), so, do in L.fwd_unpack(r):
                idx = do + np.arange(n0)[:, None, None] * d0 + np.arange(n1)[None, :, None] * d1 + np.arange(n2)
                np.add.at(seen, idx.reshape(-1), 1)
            assert (seen == 1).all()
            assert sum(L.fwd_send_splits(r)) == L.row_slab(r)
            assert sum(L.fwd_recv_splits(r)) == L.col_slab(r)


def test_block_maps_match_the_pack_descriptors():
    """SlabLayout.xmap / ymap (the addressing the fused passes use) place every element exactly
    where the fwd_pack / fwd_unpack copies put it."""
    from paper_2304_14021_b200.dist import SlabLayout
    for n, nt, P in [(33, 3, 2), (33, 2, 3), (127, 2, 8)]:
        L = SlabLayout(n, nt, P)
        for r in range(P):
            y0r, nyl = L.rows[r]
            # x map: row-slab element (t, y, x) -> send offset
            dest = np.full((nt, nyl, n), -1, dtype=np.int64)
            for (n0, n1, n2), (s0, s1), (d0, d1), so, do in L.fwd_pack(r):
                t, yy, xx = np.meshgrid(np.arange(n0), np.arange(n1), np.arange(n2), indexing="ij")
                src = so + t * s0 + yy * s1 + xx
                x = src % n
                dest[t, yy, x] = do + t * d0 + yy * d1 + xx
            for x0, cnt, off in L.xmap(r):
                t, yy, xx = np.meshgrid(np.arange(nt), np.arange(nyl), np.arange(cnt), indexing="ij")
                assert (dest[t, yy, x0 + xx] == off + (t * nyl + yy) * cnt + xx).all()
            # y map: column-slab element (t, y, c) <- receive offset
            x0r, nxl = L.cols[r]
            srcof = np.full((nt, n, nxl), -1, dtype=np.int64)
            for (n0, n1, n2), (s0, s1), (d0, d1), so, do in L.fwd_unpack(r):
                t, yy, cc = np.meshgrid(np.arange(n0), np.arange(n1), np.arange(n2), indexing="ij")
                dst = do + t * d0 + yy * d1 + cc
                srcof[t, (dst % (n * nxl)) // nxl, cc] = so + t * s0 + yy * s1 + cc
            for y0, cnt, off in L.ymap(r):
                t, yy, cc = np.meshgrid(np.arange(nt), np.arange(cnt), np.arange(nxl), indexing="ij")
                assert (srcof[t, y0 + yy, cc] == off + (t * cnt + yy) * nxl + cc).all()


@pytest.mark.parametrize("n,nt,P", [(33, 8, 2), (31, 8, 3), (129, 32, 8), (65, 4, 5), (2049, 512, 8)])
def test_library_shard_layout_equals_the_gloo_tested_layout(n, nt, P):
    """The C++ engine's slab layout (paradiag_shard_layout, csrc/shard.cu) is the one this file
    runs with real gloo collectives (dist.SlabRank, fused single-range form): same slabs, splits,
    send / receive regions and transpose-block maps for every rank — so the world-size-2 data
    movement checked against the oracle above is the library's."""
    import paper_2304_14021_b200 as pd
    from paper_2304_14021_b200 import dist

    class _Ops:
        def empty(self, count):
            return torch.zeros(1, dtype=torch.float64)

    L = dist.SlabLayout(n, nt, P)
    for r in range(P):
        got = pd.paradiag_shard_layout(n, nt, P, r)
        rk = dist.SlabRank(L, r, _Ops(), fused=True, chunks=1)
        g = rk.regions[0]
        assert (got["y0"], got["nyl"]) == L.rows[r] and (got["x0"], got["nxl"]) == L.cols[r]
        fs, fr = g["splits"]["fwd"]
        assert got["fs"] == fs and got["fr"] == fr and got["nsr"] == g["ns"]
        assert got["xm_out"] == rk.xm_out and got["ym_in"] == rk.ym_in
        assert got["ym_out"] == rk.ym_out and got["xm_in"] == rk.xm_in
