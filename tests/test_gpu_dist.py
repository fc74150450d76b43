"""Multi-rank (slab) data path on ONE GPU: P virtual ranks run the phases of
paper_2304_14021_b200/dist.py in rank order with the collectives emulated by copies
(iterate_virtual), against the single-GPU iteration (the same kernels, unsharded) and the oracle.

The sharded path differs from the single-GPU one only in which two spatial modes share a
time-pass pencil (the column slab regroups them), so the two agree to rounding; for the hinged
biharmonic twin (cond(I + ΔtA) ≈ 1e9) that is ≈ 2e-11 of max|U| on the decayed late slices, so the
bar here is 5e-11 (and 1e-10 against the oracle, the parity bar)."""
import numpy as np
import pytest

from _helpers import to_dev, rel_err
from oracle import iterate
from workloads import twin, make_u0

pytestmark = pytest.mark.gpu

CASES = {
    "c5_m128_nt32": twin("c5", m=128, nt=32),          # Neumann, 129 rows
    "c3_m128_nt32": twin("c3", m=128, nt=32),          # hinged, 127 rows
    "c5_m64_nt64": twin("c5", m=64, nt=64),
}


def _slabs(cuda_lib, p, P, fused=True, chunks=1, p2p=False):
    from paper_2304_14021_b200 import dist
    L = dist.SlabLayout(p.n, p.nt, P)
    ranks = []
    for r in range(P):
        y0, nyl = L.rows[r]
        x0, nxl = L.cols[r]
        ops = dist.GpuOps(p, 0, None, y0, nyl, x0, nxl)
        ranks.append(dist.SlabRank(L, r, ops, fused=fused, chunks=chunks, p2p=p2p))
    return L, ranks


@pytest.mark.parametrize("mode", [(True, 1, False), (False, 1, False), (True, 3, False), (True, 1, True)],
                         ids=["block-io", "pack-copies", "chunked3", "peer-stores"])
@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_virtual_ranks_match_single_gpu(cuda_lib, name, P, mode):
    fused, chunks, p2p = mode
    import torch
    from paper_2304_14021_b200 import dist
    p = CASES[name]
    u0 = make_u0(p)
    U0 = iterate.initial_iterate(p, u0)
    s = cuda_lib.Solver(p)
    U = to_dev(U0, p)
    u0d = to_dev(u0)
    L, ranks = _slabs(cuda_lib, p, P, fused, chunks, p2p)
    Us = [U.clone()[:, y0:y0 + nyl, :].contiguous().reshape(-1) for (y0, nyl) in L.rows]
    u0s = [u0d[y0:y0 + nyl, :].contiguous() for (y0, nyl) in L.rows]
    info = None
    U_o = U0
    for k in range(3):
        info = s.iterate(u0d, U, info)
        dmax, umax = dist.iterate_virtual(ranks, u0s, Us)
        U_o, io = iterate.iterate_once(p, u0, U_o)
        got = torch.cat([Us[r].reshape(p.nt, L.rows[r][1], p.n) for r in range(P)], dim=1)
        assert rel_err(got.cpu().numpy(), U.cpu().numpy()) <= 5e-11, k
        # against the oracle: as accurate as the unsharded GPU path (un-converged iterates of the
        # hinged twin carry ≈1e-9 of rounding amplification in both)
        e_single = rel_err(U.cpu().numpy(), U_o)
        assert rel_err(got.cpu().numpy(), U_o) <= max(1e-10, 1.1 * e_single), k
        assert abs(dmax - info.delta_max) <= 5e-11 * max(info.delta_max, info.u_max)
        assert abs(umax - info.u_max) <= 5e-11 * info.u_max
    for rk in ranks:
        rk.ops.close()


def test_slab_entry_points_reject_bad_geometry(cuda_lib):
    p = CASES["c5_m64_nt64"]
    with pytest.raises(cuda_lib.ParadiagError):
        cuda_lib.paradiag_init_slab(cuda_lib.make_problem(p), 0, 0, 0, 2, 0, 10)       # < 3 rows
    with pytest.raises(cuda_lib.ParadiagError):
        cuda_lib.paradiag_init_slab(cuda_lib.make_problem(p), 0, 0, 60, 10, 0, 10)     # past the grid
    q = twin("c4", m=64, nt=32)
    with pytest.raises(cuda_lib.ParadiagError):                                          # CH: replicas only
        cuda_lib.paradiag_init_slab(cuda_lib.make_problem(q), 0, 0, 0, 10, 0, 10)


def test_block_maps_and_ranges_reject_bad_arguments(cuda_lib):
    """Transpose-block maps must tile the line in order (≤ 8 blocks); slice ranges must lie in
    [0, nt); the y-range stage must be 0, 1 or 2."""
    import torch
    p = CASES["c5_m64_nt64"]
    n = p.n
    h = cuda_lib.paradiag_init_slab(cuda_lib.make_problem(p), 0, 0, 0, n, 0, n)
    try:
        a = torch.zeros(p.nt * n * n, dtype=torch.float64, device="cuda")
        b = torch.zeros_like(a)
        good = [(0, 40, 0), (40, n - 40, p.nt * n * 40)]
        cuda_lib.paradiag_slab_xpass_seg(h, a, b, False, None, good)                 # accepted
        for bad in ([(0, 40, 0), (41, n - 41, 0)],                                     # gap
                    [(0, 40, 0), (40, n - 41, 0)],                                     # does not cover
                    [(0, 40, 0), (40, 10, 0)] + [(50 + i, 1, 0) for i in range(7)] + [(57, n - 57, 0)]):  # > 8
            with pytest.raises(cuda_lib.ParadiagError):
                cuda_lib.paradiag_slab_xpass_seg(h, a, b, False, None, bad)
        with pytest.raises(cuda_lib.ParadiagError):
            cuda_lib.paradiag_slab_xrange(h, a, b, False, None, None, p.nt - 1, 2)      # past nt
        with pytest.raises(cuda_lib.ParadiagError):
            cuda_lib.paradiag_slab_yrange(h, a, b, a, 3, None, 0, 1)                   # unknown stage
        with pytest.raises(cuda_lib.ParadiagError):
            cuda_lib.paradiag_slab_update_range(h, a, b, -1, 1)
        torch.cuda.synchronize()
    finally:
        cuda_lib.paradiag_destroy(h)


def _ipc_child(handle, off, n, q):
    import torch
    import paper_2304_14021_b200 as pd
    torch.cuda.set_device(0)
    base = pd.paradiag_ipc_open(handle)
    try:
        # write through the mapped address with the library's own copy (a device kernel)
        src = torch.arange(n, dtype=torch.float64, device="cuda") + 0.5
        import ctypes
        solver = pd.Solver(twin("c5", m=64, nt=32))         # any handle: copy3d runs on its stream
        lib = pd.load()
        rc = lib.paradiag_copy3d(solver.h, ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(base + off),
                                 1, 1, n, n, n, n, n)
        torch.cuda.synchronize()
        q.put(rc)
    finally:
        pd.paradiag_ipc_close(base)


def test_ipc_export_and_map(cuda_lib):
    """The peer-memory transposes' plumbing (CUDA IPC through the C ABI): a second process maps this
    process's buffer (allocation base + the tensor's offset, as SlabRank.setup_p2p computes it) and
    stores into it with a library kernel; this process reads the values back.  Two processes on one
    device, no rank waits on another's kernels."""
    import torch
    import torch.multiprocessing as mp
    import cuda.bindings.driver as drv
    pool = torch.zeros(4096, dtype=torch.float64, device="cuda")
    t = pool[1000:1000 + 512]                          # not at the start of its allocation
    err, base, _ = drv.cuMemGetAddressRange(t.data_ptr())
    assert err == drv.CUresult.CUDA_SUCCESS
    handle = cuda_lib.paradiag_ipc_handle(int(base))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_ipc_child, args=(handle, t.data_ptr() - int(base), 512, q))
    pr.start()
    rc = q.get(timeout=300)
    pr.join(timeout=300)
    assert rc == 0 and pr.exitcode == 0
    torch.cuda.synchronize()
    assert torch.equal(t.cpu(), torch.arange(512, dtype=torch.float64) + 0.5)
    assert float(pool[:1000].abs().max()) == 0.0 and float(pool[1512:].abs().max()) == 0.0


def _nccl_world1(chunks, out_q, p2p=False):
    import os
    import socket
    import torch
    import torch.distributed as tdist
    from paper_2304_14021_b200 import dist
    import paper_2304_14021_b200 as pd
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    try:
        p = CASES["c5_m64_nt64"]
        u0 = make_u0(p)
        U0 = iterate.initial_iterate(p, u0)
        L = dist.SlabLayout(p.n, p.nt, 1)
        stream = torch.cuda.current_stream()
        ops = dist.GpuOps(p, 0, stream.cuda_stream, 0, p.n, 0, p.n)
        rk = dist.SlabRank(L, 0, ops, fused=True, chunks=chunks, self_via_comm=not p2p, p2p=p2p)
        comm = dist.TorchComm()
        if p2p:
            rk.setup_p2p(comm)            # IPC export + all_gather of the handle, NCCL fences
        U = to_dev(U0, p).reshape(-1).clone()
        u0d = to_dev(u0)
        s = pd.Solver(p)
        Ur = to_dev(U0, p)
        info = None
        errs = []
        for _ in range(3):
            rk.iterate(u0d, U, comm)
            info = s.iterate(u0d, Ur, info)
            errs.append(rel_err(U.reshape(Ur.shape).cpu().numpy(), Ur.cpu().numpy()))
        ops.close()
        out_q.put(errs)
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("chunks,p2p", [(1, False), (3, False), (1, True)], ids=["nccl", "nccl-3ranges", "p2p"])
def test_nccl_async_transposes_world1(cuda_lib, chunks, p2p):
    """A one-rank NCCL world where the kept block also goes through the (asynchronous, per slice
    range) all-to-all: the real collective's stream ordering against the library's kernels, checked
    against the unsharded iteration.  One process, one device."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_nccl_world1, args=(chunks, q, p2p))
    pr.start()
    errs = q.get(timeout=600)
    pr.join(timeout=600)
    assert pr.exitcode == 0
    assert max(errs) <= 5e-11, errs
