"""paradiag_launches_per_iteration (the bench's gpu_launches claim in --mode iterate) equals the
kernels one paradiag_iterate actually launches, counted by the library's own per-launch events
(+1 for the unprofiled k_reset_stats), on every engine path."""
import pytest

from _helpers import to_dev
from workloads import config, twin, make_u0

pytestmark = pytest.mark.gpu

PATHS = {
    "2d_fast": twin("c5", m=64, nt=32),
    "2d_ch": twin("c4", m=32, nt=16, t_window=16e-4, n_windows=1),
    "1d_penta": config("c1"),
    "1d_long_x1_unfused": twin("c6", nt=8192, t_window=8192 / 2.0 ** 20),
    "1d_long_x1_fused": twin("c6", nt=1 << 15, t_window=2.0 ** -5),
    "1d_long_rows": twin("c2", m=256, nt=8192, t_window=1.0),
    "2d_long": twin("c3", m=16, nt=8192, t_window=0.8),
}


@pytest.mark.parametrize("name", sorted(PATHS))
def test_launch_count(cuda_lib, name):
    p = PATHS[name]
    s = cuda_lib.Solver(p)
    U = s.empty()
    u0 = to_dev(make_u0(p))
    info = s.iterate(u0, U)
    s.profile(True)
    s.iterate(u0, U, info)
    prof = s.profile_read()
    assert sum(n for n, _ in prof.values()) + 1 == s.launches_per_iteration()
