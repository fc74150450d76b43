"""The multi-rank engine behind the C ABI (include/paradiag.h paradiag_init with an NCCL id,
paper_2304_14021_b200/csrc/shard.cu): slab-sharded 2D solves against the single-GPU solve and the
oracle.

* Virtual ranks (paradiag_init_virtual): P = 1, 2, 3, 8 ranks in one process on one GPU, driven
  phase by phase in rank order with the collectives emulated by device copies — the same layout,
  transpose-block maps, halos and stop rule as the NCCL path, without a multi-GPU box (and without
  ranks that wait on one another on one GPU, B200_PROFILING.md).
* A one-rank NCCL world through the C ABI: the library creates its communicator from an id it
  drew itself and all-reduces the stop-rule scalars with NCCL.
The sharded path regroups which two spatial modes share a time-pass pencil and runs the slab
kernels instead of the single-GPU ones, so it agrees with the single-GPU solve to rounding: the bar
is 5e-11 of max|U| (the hinged biharmonic twin has cond(I + ΔtA) ≈ 1e9), and 1e-10 against the
oracle (the parity bar, BASELINE.json)."""
from dataclasses import replace

import numpy as np
import pytest

from _helpers import to_dev, to_host, rel_err
from oracle import iterate
from workloads import twin, make_u0

pytestmark = pytest.mark.gpu

CASES = {
    "c5_m128_nt32": twin("c5", m=128, nt=32),          # Neumann, 129 rows, fixed K = 3 from U⁰ = 0
    "c3_m128_nt32": twin("c3", m=128, nt=32),          # hinged, 127 rows, to tol
    "c5_m64_nt64_tol": replace(twin("c5", m=64, nt=64), fixed_iters=None, init="broadcast", alpha=1e-2,
                               beta=0.1, t_window=0.05, n_windows=2),   # converging linear CH, 2 windows
}


def _solve_virtual(cuda_lib, p, P):
    import torch
    hs = cuda_lib.paradiag_init_virtual(cuda_lib.make_problem(p), P)
    try:
        rows = [cuda_lib.paradiag_local_rows(h) for h in hs]
        u0 = torch.from_numpy(np.ascontiguousarray(make_u0(p))).cuda()
        u0s = [u0[y0:y0 + n].contiguous() for y0, n in rows]
        Us = [torch.empty((p.nt, n, p.nx), dtype=torch.float64, device="cuda") for _, n in rows]
        rc, info = cuda_lib.paradiag_solve_virtual(hs, u0s, Us)
        torch.cuda.synchronize()
        return rc, info, torch.cat(Us, dim=1), rows
    finally:
        for h in hs:
            cuda_lib.paradiag_destroy(h)


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_virtual_ranks_solve_matches_single_gpu_and_oracle(cuda_lib, name, P):
    p = CASES[name]
    rc, info, U, rows = _solve_virtual(cuda_lib, p, P)
    assert [r[0] for r in rows] == sorted(r[0] for r in rows) and sum(r[1] for r in rows) == p.ny
    s = cuda_lib.Solver(p)
    V = s.empty()
    rc1, info1 = s.solve(to_dev(make_u0(p)), V)
    assert rc == rc1 and list(info.iters[:p.n_windows]) == list(info1.iters[:p.n_windows])
    assert info.diverging == info1.diverging
    assert rel_err(to_host(U), to_host(V)) <= 5e-11
    U_o, iters_o, _, _ = iterate.solve(p, make_u0(p))
    assert list(info.iters[:p.n_windows]) == iters_o
    assert rel_err(to_host(U), U_o) <= 1e-10


@pytest.mark.parametrize("P", [2, 3])
def test_virtual_ranks_iterate_reports_global_norms(cuda_lib, P):
    """paradiag_iterate_virtual: one defect-correction step per call; ‖δ‖∞ and ‖U‖∞ are the maxima
    over the ranks (the all-reduce) and equal the single-GPU iteration's."""
    import torch
    p = CASES["c3_m128_nt32"]
    hs = cuda_lib.paradiag_init_virtual(cuda_lib.make_problem(p), P)
    try:
        rows = [cuda_lib.paradiag_local_rows(h) for h in hs]
        u0 = to_dev(make_u0(p))
        U0 = to_dev(iterate.initial_iterate(p, make_u0(p)), p)
        Us = [U0[:, y0:y0 + n].contiguous() for y0, n in rows]
        u0s = [u0[y0:y0 + n].contiguous() for y0, n in rows]
        s = cuda_lib.Solver(p)
        V = U0.clone()
        a = b = None
        for k in range(3):
            a = cuda_lib.paradiag_iterate_virtual(hs, u0s, Us, a)
            b = s.iterate(u0, V, b)
            assert a.iters == b.iters == k + 1
            # (relative to ‖U‖∞: by iteration 3 the increment of c3 is at rounding level, 1e-15)
            assert abs(a.delta_max - b.delta_max) <= 1e-11 * max(b.delta_max, 1e-3 * b.u_max)
            assert abs(a.u_max - b.u_max) <= 1e-12 * b.u_max
        assert rel_err(to_host(torch.cat(Us, dim=1)), to_host(V)) <= 5e-11
    finally:
        for h in hs:
            cuda_lib.paradiag_destroy(h)


def test_nccl_one_rank_world_through_the_abi(cuda_lib):
    """paradiag_nccl_unique_id + paradiag_init(…, id, 0, 1): the library owns an NCCL communicator
    and the sharded solve (NCCL all-reduce of the stop rule) equals the single-GPU solve."""
    p = CASES["c3_m128_nt32"]
    nid = cuda_lib.paradiag_nccl_unique_id()
    assert len(nid) == 128
    sh = cuda_lib.Solver(p, nccl_id=nid, rank=0, nranks=1)
    assert (sh.y0, sh.ny) == (0, p.ny)
    U = sh.empty()
    rc, info = sh.solve(to_dev(make_u0(p)), U)
    s = cuda_lib.Solver(p)
    V = s.empty()
    rc1, info1 = s.solve(to_dev(make_u0(p)), V)
    assert rc == rc1 == 0 and info.iters[0] == info1.iters[0]
    assert rel_err(to_host(U), to_host(V)) <= 5e-11
    # P_α⁻¹ on the (whole) slab through the sharded handle
    r = np.random.default_rng(3).uniform(-1, 1, (p.nt, p.ny, p.nx))
    d1, d2 = sh.empty(), s.empty()
    sh.apply_precond(to_dev(r), d1)
    s.apply_precond(to_dev(r), d2)
    assert rel_err(to_host(d1), to_host(d2)) <= 1e-12
    sh.close()


def test_sharded_handle_rejects_unsupported(cuda_lib):
    nid = cuda_lib.paradiag_nccl_unique_id()
    with pytest.raises(cuda_lib.ParadiagError):        # CH runs as replicas
        cuda_lib.Solver(twin("c4", m=64, nt=32, t_window=32e-4, n_windows=1), nccl_id=nid, rank=0, nranks=1)
    with pytest.raises(cuda_lib.ParadiagError):        # rank outside [0, nranks)
        cuda_lib.Solver(CASES["c3_m128_nt32"], nccl_id=nid, rank=2, nranks=2)
    with pytest.raises(cuda_lib.ParadiagError):        # nranks > 1 without an id
        cuda_lib.Solver(CASES["c3_m128_nt32"], nranks=2)
