"""The device-side window loop (CUDA graph with a conditional WHILE node around one iteration,
paradiag_solve's default) against the host loop (PARADIAG_GRAPH=0): the same kernels in the same
order, so iteration counts, convergence flags and iterates agree exactly, on every engine path."""
import numpy as np
import pytest

from _helpers import to_dev, to_host
from workloads import config, twin, make_u0

pytestmark = pytest.mark.gpu

PATHS = {
    "c1": config("c1"),
    "c2_small": twin("c2", m=37, nt=8),
    "c3_m32": twin("c3", m=32, nt=16),
    "c4_m32_2win": twin("c4", m=32, nt=16, t_window=16e-4, n_windows=2),
    "c4e_m16": twin("c4e", m=16, nt=8, t_window=8e-4, n_windows=2),
    "c5_m64_K3": twin("c5", m=64, nt=32),
    "c6_nt8192": twin("c6", nt=8192, t_window=8192 / 2.0 ** 20),
    "maxiter_hit": twin("c3", m=32, nt=16, max_iter=2),
}


@pytest.mark.parametrize("name", sorted(PATHS))
def test_graph_loop_equals_host_loop(cuda_lib, monkeypatch, name):
    p = PATHS[name]
    u0 = to_dev(make_u0(p))
    out = []
    for g in ("1", "0"):
        monkeypatch.setenv("PARADIAG_GRAPH", g)
        s = cuda_lib.Solver(p)
        U = s.empty()
        rc, info = s.solve(u0, U)
        out.append((rc, list(info.iters[:p.n_windows]), info.converged, list(info.last_rel[:p.n_windows]),
                    to_host(U)))
        s.close()
    (rc_g, it_g, cv_g, rel_g, U_g), (rc_h, it_h, cv_h, rel_h, U_h) = out
    assert rc_g == rc_h and it_g == it_h and cv_g == cv_h
    assert np.array_equal(U_g, U_h)
    assert rel_g == rel_h


def test_graph_loop_repeated_and_new_buffer(cuda_lib):
    """The captured graph is reused for the same U and re-captured for another."""
    p = twin("c3", m=32, nt=16)
    u0 = to_dev(make_u0(p))
    s = cuda_lib.Solver(p)
    U1, U2 = s.empty(), s.empty()
    r1 = s.solve(u0, U1)
    r2 = s.solve(u0, U1)
    r3 = s.solve(u0, U2)
    assert list(r1[1].iters[:1]) == list(r2[1].iters[:1]) == list(r3[1].iters[:1])
    assert np.array_equal(to_host(U1), to_host(U2))
