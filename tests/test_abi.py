"""C-ABI library: loads, exports every symbol include/paradiag.h declares, validates problems
on the host.  No compute calls (no GPU needed)."""
import ctypes
import os
import re

import pytest

import paper_2304_14021_b200 as pd
from workloads import config, CONFIGS

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "paradiag.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2304_14021_b200 import build
    build.build()
    return pd.load()


def test_exports_every_declared_symbol(lib):
    decl = set(re.findall(r"\b(paradiag_\w+)\s*\(", open(HDR).read()))
    assert len(decl) >= 12
    for name in decl:
        assert hasattr(lib, name), name
    assert set(pd.EXPORTS) == decl


def test_abi_version_and_strerror(lib):
    assert lib.paradiag_abi_version() == pd.ABI_VERSION == 5
    assert pd.strerror(pd.PD_EINVAL).startswith("PD_EINVAL")
    assert pd.strerror(pd.PD_ESINGULAR).startswith("PD_ESINGULAR")


def test_struct_layout_matches_header():
    # pd_problem: 4 int32, int64, 8 doubles, 6 int32 -> 112 bytes with natural alignment
    assert ctypes.sizeof(pd.pd_problem) == 112
    assert ctypes.sizeof(pd.pd_iter_info) == 48 + 8            # + int32 growth, padded to 8
    assert ctypes.sizeof(pd.pd_solve_info) == 8 + 64 * 4 + 64 * 8 + 8 + 8   # + int32 diverging, padded


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_workspace_bytes_all_configs(lib, name):
    b = pd.paradiag_workspace_bytes(pd.make_problem(config(name)))
    p = config(name)
    assert b >= p.dofs * 8


@pytest.mark.parametrize("bad", [dict(alpha=0.0), dict(alpha=1.0), dict(nt=96), dict(nt=3000), dict(nt=1), dict(nt=1 << 21),
                                 dict(theta=0.4), dict(theta=1.1), dict(m=100), dict(eps=-1.0), dict(t_window=0.0),
                                 dict(kind="cahn_hilliard"), dict(n_windows=0), dict(tol=0.0)])
def test_invalid_problems_rejected(lib, bad):
    p = pd.make_problem(config("c3"), **bad)
    with pytest.raises(pd.ParadiagError) as e:
        pd.paradiag_workspace_bytes(p)
    assert e.value.code == pd.PD_EINVAL


def test_max_nt_accepted(lib):
    """N_t = 4096 is the documented maximum (include/paradiag.h); the GPU parity suite runs it."""
    assert pd.paradiag_workspace_bytes(pd.make_problem(config("c2"), nt=4096)) > 0


def test_time_avg_jacobian_is_a_ch_option(lib):
    """NEXT-4: the time-averaged Jacobian applies to the CH kinds only."""
    assert pd.paradiag_workspace_bytes(pd.make_problem(config("c4t"))) > \
        pd.paradiag_workspace_bytes(pd.make_problem(config("c4")))
    with pytest.raises(pd.ParadiagError):
        pd.paradiag_workspace_bytes(pd.make_problem(config("c3"), jacobian="time_avg"))
    with pytest.raises(pd.ParadiagError):
        pd.paradiag_workspace_bytes(pd.make_problem(config("c4"), jacobian=7))


def test_long_window_limits(lib):
    """N_t > 4096 takes the four-step time pass (k_tlong.cuh): up to 2^20 (c6, NEXT-3); in 1D it
    solves Step (2) in the DST/DCT eigenbasis, so m must be a power of two there."""
    b = pd.paradiag_workspace_bytes(pd.make_problem(config("c6")))
    p = config("c6")
    assert b >= 3 * p.dofs * 8                       # U-sized work + Y + X (complex, ⌈N_s/2⌉ pairs each)
    with pytest.raises(pd.ParadiagError):
        pd.paradiag_workspace_bytes(pd.make_problem(config("c6"), m=100))
    assert pd.paradiag_workspace_bytes(pd.make_problem(config("c6"), m=100, nt=4096)) > 0


def test_theta_half_accepted_but_not_for_ch(lib):
    """θ-method: θ ∈ [1/2, 1] for the linear kinds; CH PinT-I is backward Euler."""
    assert pd.paradiag_workspace_bytes(pd.make_problem(config("c3"), theta=0.5)) > 0
    with pytest.raises(pd.ParadiagError):
        pd.paradiag_workspace_bytes(pd.make_problem(config("c4"), theta=0.5))


def test_ch_requires_2d_neumann(lib):
    p = pd.make_problem(config("c4"), dim=1)
    with pytest.raises(pd.ParadiagError):
        pd.paradiag_workspace_bytes(p)


def test_init_without_device_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    rc = lib.paradiag_init(ctypes.byref(pd.make_problem(config("c1"))), 0, None, None, 0, 1, ctypes.byref(h))
    assert rc == pd.PD_ECUDA and not h.value


def test_sharded_init_validates_before_any_collective(lib):
    """paradiag_init with nranks > 1 rejects unsupported problems / ranks with PD_EINVAL before it
    touches CUDA or NCCL (no rank ever blocks in the communicator set-up on a bad call)."""
    h = ctypes.c_void_p()
    nid = b"\0" * 128
    for p, rank, nranks in ((pd.make_problem(config("c4")), 0, 2),                 # CH: replicas only
                            (pd.make_problem(config("c3")), 3, 2),                 # rank outside the world
                            (pd.make_problem(config("c3")), 0, 9),                 # more than 8 ranks
                            (pd.make_problem(config("c3"), m=8), 0, 4)):           # < 3 rows per rank
        rc = lib.paradiag_init(ctypes.byref(p), 0, None, nid, rank, nranks, ctypes.byref(h))
        assert rc == pd.PD_EINVAL and not h.value


def test_workspace_bytes_per_rank(lib):
    one = pd.paradiag_workspace_bytes(pd.make_problem(config("c5")))
    eight = pd.paradiag_workspace_bytes(pd.make_problem(config("c5")), 8)
    assert eight < one


@pytest.mark.parametrize("nt", [100, 625, 1000, 10 ** 4, 40000, 10 ** 6])
def test_mixed_radix_windows_accepted(lib, nt):
    """N_t = 2^a 5^b (the paper's 10^4; 40000; 10^6) takes the mixed-radix
    long-window path."""
    from dataclasses import replace
    assert pd.paradiag_workspace_bytes(pd.make_problem(replace(config("c6n"), nt=nt))) > 0
