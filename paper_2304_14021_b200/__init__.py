"""Python binding of libparadiag.so (include/paradiag.h) — argument marshalling only.

Every step of the ParaDiag hot path runs in the sm_100a kernels behind the C ABI; this module
converts torch CUDA tensors to device pointers and calls the entry points of the same names.
There is no CPU fallback: if the shared library is missing or the device is not an sm_100a
B200, calls raise ``ParadiagError``.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libparadiag.so")

PD_OK, PD_NOT_CONVERGED = 0, 1
PD_EINVAL, PD_ESINGULAR, PD_ECUDA, PD_ENCCL, PD_ENOMEM, PD_EDIVERGED = -1, -2, -3, -4, -5, -6
KINDS = {"biharmonic": 0, "linear_ch": 1, "cahn_hilliard": 2, "cahn_hilliard_eyre": 3}
BCS = {"neumann": 0, "hinged": 1}
INITS = {"broadcast": 0, "zero": 1}
JACOBIANS = {"scalar": 0, "time_avg": 1}
MAX_WINDOWS = 64


class ParadiagError(RuntimeError):
    def __init__(self, code, where, detail=""):
        self.code = code
        super().__init__(f"{where}: {strerror(code)} ({detail})")


class pd_problem(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("bc", ctypes.c_int32), ("dim", ctypes.c_int32),
                ("nt", ctypes.c_int32), ("m", ctypes.c_int64), ("t_window", ctypes.c_double),
                ("alpha", ctypes.c_double), ("theta", ctypes.c_double), ("beta", ctypes.c_double),
                ("eps", ctypes.c_double), ("tol", ctypes.c_double), ("omega", ctypes.c_double),
                ("tau", ctypes.c_double), ("n_windows", ctypes.c_int32), ("max_iter", ctypes.c_int32),
                ("fixed_iters", ctypes.c_int32), ("init", ctypes.c_int32), ("jacobian", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class pd_iter_info(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("converged", ctypes.c_int32), ("delta_max", ctypes.c_double),
                ("u_max", ctypes.c_double), ("rel", ctypes.c_double), ("jbar", ctypes.c_double),
                ("omega", ctypes.c_double), ("growth", ctypes.c_int32)]


class pd_solve_info(ctypes.Structure):
    _fields_ = [("windows_done", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("iters", ctypes.c_int32 * MAX_WINDOWS), ("last_rel", ctypes.c_double * MAX_WINDOWS),
                ("seconds", ctypes.c_double), ("diverging", ctypes.c_int32)]


class pd_kernel_time(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_int32), ("total_ms", ctypes.c_double)]


_lib = None
EXPORTS = ["paradiag_profile", "paradiag_profile_read", "paradiag_abi_version", "paradiag_strerror", "paradiag_last_error", "paradiag_workspace_bytes",
           "paradiag_init", "paradiag_residual", "paradiag_apply_precond", "paradiag_apply_precond_jt", "paradiag_iterate",
           "paradiag_solve", "paradiag_solve_host", "paradiag_launches_per_iteration", "paradiag_destroy",
           "paradiag_init_slab", "paradiag_slab_geometry", "paradiag_slab_residual", "paradiag_slab_xpass",
           "paradiag_slab_ypass", "paradiag_slab_xpass_seg", "paradiag_slab_ypass_seg", "paradiag_slab_xrange", "paradiag_slab_yrange",
           "paradiag_slab_update_range", "paradiag_ipc_handle", "paradiag_ipc_open", "paradiag_ipc_close",
           "paradiag_slab_update", "paradiag_copy3d", "paradiag_stats_reset",
           "paradiag_stats_read", "paradiag_tslab_pitch", "paradiag_tslab_residual", "paradiag_tslab_time",
           "paradiag_tslab_update", "paradiag_nccl_unique_id", "paradiag_local_rows", "paradiag_init_virtual",
           "paradiag_iterate_virtual", "paradiag_solve_virtual", "paradiag_shard_layout"]
ABI_VERSION = 5
GROWTH_LIMIT = 3          # PD_GROWTH_LIMIT


def load(path: str = LIB_PATH):
    """Load libparadiag.so (built by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ParadiagError(PD_ECUDA, "load", f"{path} not built; run python paper_2304_14021_b200/build.py")
    lib = ctypes.CDLL(path)
    vp, P = ctypes.c_void_p, ctypes.POINTER
    lib.paradiag_abi_version.restype = ctypes.c_int
    lib.paradiag_strerror.restype = ctypes.c_char_p
    lib.paradiag_strerror.argtypes = [ctypes.c_int]
    lib.paradiag_last_error.restype = ctypes.c_char_p
    lib.paradiag_workspace_bytes.argtypes = [P(pd_problem), ctypes.c_int, P(ctypes.c_size_t)]
    lib.paradiag_init.argtypes = [P(pd_problem), ctypes.c_int, vp, ctypes.c_char_p, ctypes.c_int, ctypes.c_int, P(vp)]
    lib.paradiag_nccl_unique_id.argtypes = [ctypes.c_char_p]
    lib.paradiag_local_rows.argtypes = [vp, P(ctypes.c_int64), P(ctypes.c_int64)]
    lib.paradiag_init_virtual.argtypes = [P(pd_problem), ctypes.c_int, vp, ctypes.c_int, P(vp)]
    lib.paradiag_iterate_virtual.argtypes = [P(vp), ctypes.c_int, P(vp), P(vp), P(pd_iter_info)]
    lib.paradiag_solve_virtual.argtypes = [P(vp), ctypes.c_int, P(vp), P(vp), P(pd_solve_info)]
    lib.paradiag_shard_layout.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, P(ctypes.c_int64),
                                          ctypes.c_int64]
    lib.paradiag_residual.argtypes = [vp, vp, vp, vp, P(ctypes.c_double)]
    lib.paradiag_apply_precond.argtypes = [vp, vp, vp, ctypes.c_double]
    lib.paradiag_apply_precond_jt.argtypes = [vp, vp, vp, vp]
    lib.paradiag_iterate.argtypes = [vp, vp, vp, P(pd_iter_info)]
    lib.paradiag_solve.argtypes = [vp, vp, vp, P(pd_solve_info)]
    lib.paradiag_solve_host.argtypes = [vp, vp, vp, P(pd_solve_info)]
    lib.paradiag_launches_per_iteration.argtypes = [vp]
    lib.paradiag_profile.argtypes = [vp, ctypes.c_int]
    lib.paradiag_profile_read.argtypes = [vp, P(pd_kernel_time), ctypes.c_int, P(ctypes.c_int)]
    lib.paradiag_destroy.argtypes = [vp]
    lib.paradiag_destroy.restype = None
    i64 = ctypes.c_int64
    lib.paradiag_init_slab.argtypes = [P(pd_problem), ctypes.c_int, vp, i64, i64, i64, i64, P(vp)]
    lib.paradiag_slab_geometry.argtypes = [vp, P(i64), P(i64), P(i64), P(i64)]
    lib.paradiag_slab_residual.argtypes = [vp, vp, vp, vp, vp, vp]
    lib.paradiag_slab_xpass.argtypes = [vp, vp, vp, ctypes.c_int]
    lib.paradiag_slab_ypass.argtypes = [vp, vp]
    lib.paradiag_slab_xpass_seg.argtypes = [vp, vp, vp, ctypes.c_int, vp, vp]
    lib.paradiag_slab_ypass_seg.argtypes = [vp, vp, vp, vp, vp, vp]
    lib.paradiag_slab_xrange.argtypes = [vp, vp, vp, ctypes.c_int, vp, vp, i64, i64]
    lib.paradiag_slab_yrange.argtypes = [vp, vp, vp, vp, ctypes.c_int, vp, i64, i64]
    lib.paradiag_slab_update_range.argtypes = [vp, vp, vp, i64, i64]
    lib.paradiag_ipc_handle.argtypes = [vp, ctypes.c_char_p]
    lib.paradiag_ipc_open.argtypes = [ctypes.c_char_p, P(vp)]
    lib.paradiag_ipc_close.argtypes = [vp]
    lib.paradiag_slab_update.argtypes = [vp, vp, vp]
    lib.paradiag_copy3d.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, i64]
    lib.paradiag_stats_reset.argtypes = [vp]
    lib.paradiag_stats_read.argtypes = [vp, P(ctypes.c_double), P(ctypes.c_double)]
    lib.paradiag_tslab_pitch.argtypes = [vp, P(i64)]
    lib.paradiag_tslab_residual.argtypes = [vp, vp, vp, i64, vp, i64]
    lib.paradiag_tslab_time.argtypes = [vp, vp, i64, i64]
    lib.paradiag_tslab_update.argtypes = [vp, vp, i64, vp, i64]
    for name in EXPORTS:
        if name not in ("paradiag_destroy",):
            getattr(lib, name).restype = getattr(lib, name).restype or ctypes.c_int
    if lib.paradiag_abi_version() != ABI_VERSION:
        raise ParadiagError(PD_ECUDA, "load", "ABI version mismatch")
    _lib = lib
    return lib


def strerror(code: int) -> str:
    try:
        return load().paradiag_strerror(code).decode()
    except Exception:  # library missing: still name the code
        return f"status {code}"


def _check(rc, where):
    if rc < 0:
        raise ParadiagError(rc, where, load().paradiag_last_error().decode())
    return rc


def make_problem(obj=None, **kw) -> pd_problem:
    """pd_problem from keyword arguments or from any object carrying the same field names
    (e.g. workloads.Problem).  kind/bc/init accept the names in KINDS/BCS/INITS."""
    f = {}
    if obj is not None:
        for k in ("kind", "bc", "dim", "nt", "m", "t_window", "alpha", "theta", "beta", "eps", "tol",
                  "omega", "tau", "n_windows", "max_iter", "fixed_iters", "init", "jacobian"):
            if hasattr(obj, k):
                f[k] = getattr(obj, k)
    f.update(kw)
    p = pd_problem()
    p.kind = KINDS[f["kind"]] if isinstance(f["kind"], str) else int(f["kind"])
    p.bc = BCS[f["bc"]] if isinstance(f["bc"], str) else int(f["bc"])
    p.dim = int(f["dim"])
    p.nt = int(f["nt"])
    p.m = int(f["m"])
    p.t_window = float(f["t_window"])
    p.alpha = float(f["alpha"])
    p.theta = float(f.get("theta", 1.0))
    p.beta = float(f.get("beta", 0.0))
    p.eps = float(f.get("eps", 0.0))
    p.tol = float(f.get("tol", 1e-10))
    p.omega = float(f.get("omega", 1.0))
    tau = f.get("tau", float("inf"))
    p.tau = float(tau) if tau is not None else float("inf")
    p.n_windows = int(f.get("n_windows", 1))
    p.max_iter = int(f.get("max_iter", 100))
    fi = f.get("fixed_iters")
    p.fixed_iters = int(fi) if fi else 0
    init = f.get("init", "broadcast")
    p.init = INITS[init] if isinstance(init, str) else int(init)
    jac = f.get("jacobian", "scalar")
    p.jacobian = JACOBIANS[jac] if isinstance(jac, str) else int(jac)
    p.reserved = 0
    return p


def _ptr(t, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise ParadiagError(PD_EINVAL, name, "expected a contiguous float64 CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def _check_tensor(t, name, numel, device):
    """The C ABI receives raw pointers: refuse a tensor of the wrong size or on another device
    before the library would read or write out of bounds."""
    _ptr(t, name)
    if t.numel() != numel:
        raise ParadiagError(PD_EINVAL, name, f"has {t.numel()} elements, expected {numel}")
    if t.device.index != device:
        raise ParadiagError(PD_EINVAL, name, f"is on cuda:{t.device.index}, the handle on cuda:{device}")
    return t


# ---------------------------------------------------------------- thin C-ABI mirrors
def paradiag_workspace_bytes(problem: pd_problem, nranks: int = 1) -> int:
    b = ctypes.c_size_t(0)
    _check(load().paradiag_workspace_bytes(ctypes.byref(problem), int(nranks), ctypes.byref(b)),
           "paradiag_workspace_bytes")
    return b.value


def paradiag_init(problem: pd_problem, device: int = 0, stream=None, nccl_id: bytes = None, rank: int = 0,
                  nranks: int = 1) -> ctypes.c_void_p:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device).cuda_stream
    if nccl_id is not None and len(nccl_id) != 128:
        raise ParadiagError(PD_EINVAL, "paradiag_init", "nccl_id must be 128 bytes")
    h = ctypes.c_void_p()
    _check(load().paradiag_init(ctypes.byref(problem), int(device), ctypes.c_void_p(stream), nccl_id, int(rank),
                                int(nranks), ctypes.byref(h)), "paradiag_init")
    return h


def paradiag_nccl_unique_id() -> bytes:
    """128-byte NCCL id for a sharded paradiag_init (rank 0 only; broadcast it)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().paradiag_nccl_unique_id(buf), "paradiag_nccl_unique_id")
    return buf.raw


def paradiag_shard_layout(n: int, nt: int, nranks: int, rank: int) -> dict:
    """The sharded engine's layout of one rank (host only): slabs, splits and transpose-block maps."""
    P = nranks
    cap = 6 + 4 * P + 4 * (1 + 3 * P)
    buf = (ctypes.c_int64 * cap)()
    _check(load().paradiag_shard_layout(int(n), int(nt), int(nranks), int(rank), buf, cap), "paradiag_shard_layout")
    v = list(buf)
    out = dict(zip(("y0", "nyl", "x0", "nxl", "nsr", "so"), v[:6]))
    k = 6
    for name in ("fs", "fr", "cfs", "cfr"):
        out[name] = v[k:k + P]
        k += P
    for name in ("xm_out", "ym_in", "ym_out", "xm_in"):
        blk = v[k + 1:k + 1 + 3 * P]
        out[name] = [tuple(blk[3 * i:3 * i + 3]) for i in range(P)]
        k += 1 + 3 * P
    return out


def paradiag_local_rows(h):
    y0, n = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(load().paradiag_local_rows(h, ctypes.byref(y0), ctypes.byref(n)), "paradiag_local_rows")
    return y0.value, n.value


def paradiag_init_virtual(problem: pd_problem, nranks: int, device: int = 0, stream=None):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device).cuda_stream
    hs = (ctypes.c_void_p * nranks)()
    _check(load().paradiag_init_virtual(ctypes.byref(problem), int(device), ctypes.c_void_p(stream), int(nranks), hs),
           "paradiag_init_virtual")
    return [ctypes.c_void_p(h) for h in hs]


def _ptr_array(ts, name):
    return (ctypes.c_void_p * len(ts))(*[_ptr(t, name).value for t in ts])


def paradiag_iterate_virtual(hs, u0s, Us, info: pd_iter_info = None) -> pd_iter_info:
    info = info or pd_iter_info()
    arr = (ctypes.c_void_p * len(hs))(*[h.value for h in hs])
    _check(load().paradiag_iterate_virtual(arr, len(hs), _ptr_array(u0s, "u0_l"), _ptr_array(Us, "U_l"),
                                           ctypes.byref(info)), "paradiag_iterate_virtual")
    return info


def paradiag_solve_virtual(hs, u0s, Us):
    info = pd_solve_info()
    arr = (ctypes.c_void_p * len(hs))(*[h.value for h in hs])
    rc = _check(load().paradiag_solve_virtual(arr, len(hs), _ptr_array(u0s, "u0_l"), _ptr_array(Us, "U_l"),
                                              ctypes.byref(info)), "paradiag_solve_virtual")
    return rc, info


def paradiag_residual(h, u0, U, r, want_jbar=False):
    j = ctypes.c_double(0.0)
    _check(load().paradiag_residual(h, _ptr(u0, "u0"), _ptr(U, "U"), _ptr(r, "r"),
                                    ctypes.byref(j) if want_jbar else None), "paradiag_residual")
    return j.value


def paradiag_apply_precond(h, r, delta, jbar: float = 0.0):
    _check(load().paradiag_apply_precond(h, _ptr(r, "r"), _ptr(delta, "delta"), float(jbar)),
           "paradiag_apply_precond")


def paradiag_apply_precond_jt(h, r, delta, jt):
    """δ = G̃'⁻¹ r with the time-averaged Jacobian diag(jt) (NEXT-4); returns the status (1: the
    inner GMRES hit its cap)."""
    return _check(load().paradiag_apply_precond_jt(h, _ptr(r, "r"), _ptr(delta, "delta"), _ptr(jt, "jt")),
                  "paradiag_apply_precond_jt")


def paradiag_iterate(h, u0, U, info: pd_iter_info = None) -> pd_iter_info:
    info = info or pd_iter_info()
    _check(load().paradiag_iterate(h, _ptr(u0, "u0"), _ptr(U, "U"), ctypes.byref(info)), "paradiag_iterate")
    return info


def paradiag_solve(h, u0, U):
    info = pd_solve_info()
    rc = _check(load().paradiag_solve(h, _ptr(u0, "u0"), _ptr(U, "U"), ctypes.byref(info)), "paradiag_solve")
    return rc, info


def paradiag_solve_host(h, u0_host: np.ndarray, uT_host: np.ndarray):
    for a in (u0_host, uT_host):
        if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
            raise ParadiagError(PD_EINVAL, "paradiag_solve_host", "host arrays must be contiguous float64")
    info = pd_solve_info()
    rc = _check(load().paradiag_solve_host(h, u0_host.ctypes.data_as(ctypes.c_void_p),
                                           uT_host.ctypes.data_as(ctypes.c_void_p), ctypes.byref(info)),
                "paradiag_solve_host")
    return rc, info


def paradiag_launches_per_iteration(h) -> int:
    return load().paradiag_launches_per_iteration(h)


def paradiag_profile(h, enable: bool = True):
    _check(load().paradiag_profile(h, 1 if enable else 0), "paradiag_profile")


def paradiag_profile_read(h) -> dict:
    """{kernel name: (launches, total_ms)} accumulated since paradiag_profile(h, True)."""
    n = ctypes.c_int(0)
    buf = (pd_kernel_time * 32)()
    _check(load().paradiag_profile_read(h, buf, 32, ctypes.byref(n)), "paradiag_profile_read")
    return {buf[i].name.decode(): (buf[i].launches, buf[i].total_ms) for i in range(min(n.value, 32))}


def paradiag_init_slab(problem: pd_problem, device: int, stream, y0: int, nyl: int, x0: int, nxl: int):
    h = ctypes.c_void_p()
    _check(load().paradiag_init_slab(ctypes.byref(problem), int(device), ctypes.c_void_p(stream), int(y0), int(nyl),
                                     int(x0), int(nxl), ctypes.byref(h)), "paradiag_init_slab")
    return h


def _optr(t, name):
    return ctypes.c_void_p(None) if t is None else _ptr(t, name)


def paradiag_slab_residual(h, u0_l, U_l, halo_lo, halo_hi, r_l):
    _check(load().paradiag_slab_residual(h, _ptr(u0_l, "u0_l"), _ptr(U_l, "U_l"), _optr(halo_lo, "halo_lo"),
                                         _optr(halo_hi, "halo_hi"), _ptr(r_l, "r_l")), "paradiag_slab_residual")


def paradiag_slab_xpass(h, src, dst, want_dmax=False):
    _check(load().paradiag_slab_xpass(h, _ptr(src, "in"), _ptr(dst, "out"), 1 if want_dmax else 0),
           "paradiag_slab_xpass")


def paradiag_slab_ypass(h, cols):
    _check(load().paradiag_slab_ypass(h, _ptr(cols, "cols")), "paradiag_slab_ypass")


def _segmap(seg):
    """[(e0, cnt, off), ...] -> int64 {k, e0, cnt, off, ...} (None: slab layout)."""
    if seg is None:
        return None, None
    a = np.array([len(seg)] + [v for blk in seg for v in blk], dtype=np.int64)
    return a, a.ctypes.data_as(ctypes.c_void_p)


def paradiag_slab_xpass_seg(h, src, dst, want_dmax=False, seg_in=None, seg_out=None):
    a_in, p_in = _segmap(seg_in)
    a_out, p_out = _segmap(seg_out)
    _check(load().paradiag_slab_xpass_seg(h, _ptr(src, "src"), _ptr(dst, "dst"), int(bool(want_dmax)), p_in, p_out),
           "paradiag_slab_xpass_seg")


def paradiag_slab_ypass_seg(h, src, cols, dst, seg_in=None, seg_out=None):
    a_in, p_in = _segmap(seg_in)
    a_out, p_out = _segmap(seg_out)
    _check(load().paradiag_slab_ypass_seg(h, _ptr(src, "src"), _ptr(cols, "cols"), _ptr(dst, "dst"), p_in, p_out),
           "paradiag_slab_ypass_seg")


def paradiag_slab_xrange(h, src, dst, want_dmax, seg_in, seg_out, n0, nn):
    a_in, p_in = _segmap(seg_in)
    a_out, p_out = _segmap(seg_out)
    _check(load().paradiag_slab_xrange(h, _ptr(src, "src"), _ptr(dst, "dst"), int(bool(want_dmax)), p_in, p_out,
                                       int(n0), int(nn)), "paradiag_slab_xrange")


def paradiag_slab_yrange(h, src, cols, dst, stage, seg, n0, nn):
    a, pp = _segmap(seg)
    _check(load().paradiag_slab_yrange(h, _ptr(src, "src"), _ptr(cols, "cols"), _ptr(dst, "dst"), int(stage), pp,
                                       int(n0), int(nn)), "paradiag_slab_yrange")


def paradiag_slab_update_range(h, U_l, delta_l, n0, nn):
    _check(load().paradiag_slab_update_range(h, _ptr(U_l, "U_l"), _ptr(delta_l, "delta_l"), int(n0), int(nn)),
           "paradiag_slab_update_range")


def paradiag_ipc_handle(addr) -> bytes:
    """64-byte CUDA IPC handle of the allocation containing device address addr (int or tensor)."""
    if not isinstance(addr, int):
        addr = addr.data_ptr()
    buf = ctypes.create_string_buffer(64)
    _check(load().paradiag_ipc_handle(ctypes.c_void_p(addr), buf), "paradiag_ipc_handle")
    return buf.raw


def paradiag_ipc_open(handle: bytes) -> int:
    """Map a peer's exported allocation; returns its device address in this process."""
    ptr = ctypes.c_void_p()
    _check(load().paradiag_ipc_open(ctypes.c_char_p(handle), ctypes.byref(ptr)), "paradiag_ipc_open")
    return int(ptr.value)


def paradiag_ipc_close(ptr: int):
    _check(load().paradiag_ipc_close(ctypes.c_void_p(ptr)), "paradiag_ipc_close")


def paradiag_slab_update(h, U_l, delta_l):
    _check(load().paradiag_slab_update(h, _ptr(U_l, "U_l"), _ptr(delta_l, "delta_l")), "paradiag_slab_update")


def paradiag_copy3d(h, src, dst, n, s, d, src_off=0, dst_off=0):
    """dst[dst_off + a*d[0] + b*d[1] + c] = src[src_off + a*s[0] + b*s[1] + c], (a, b, c) < n.
    src/dst are flat float64 CUDA tensors; offsets and strides in elements."""
    import torch
    for t, nm in ((src, "src"), (dst, "dst")):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
            raise ParadiagError(PD_EINVAL, nm, "expected a contiguous float64 CUDA tensor")
    sp = ctypes.c_void_p(src.data_ptr() + 8 * int(src_off))
    dp = ctypes.c_void_p(dst.data_ptr() + 8 * int(dst_off))
    _check(load().paradiag_copy3d(h, sp, dp, int(n[0]), int(n[1]), int(n[2]), int(s[0]), int(s[1]), int(d[0]),
                                  int(d[1])), "paradiag_copy3d")


def paradiag_stats_reset(h):
    _check(load().paradiag_stats_reset(h), "paradiag_stats_reset")


def paradiag_stats_read(h):
    a, b = ctypes.c_double(0.0), ctypes.c_double(0.0)
    _check(load().paradiag_stats_read(h, ctypes.byref(a), ctypes.byref(b)), "paradiag_stats_read")
    return a.value, b.value


def paradiag_tslab_pitch(h) -> int:
    v = ctypes.c_int64(0)
    _check(load().paradiag_tslab_pitch(h, ctypes.byref(v)), "paradiag_tslab_pitch")
    return v.value


def paradiag_tslab_residual(h, u_prev, U_l, nn, blocks, bcols):
    _check(load().paradiag_tslab_residual(h, _ptr(u_prev, "u_prev"), _ptr(U_l, "U_l"), int(nn), _ptr(blocks, "blocks"),
                                          int(bcols)), "paradiag_tslab_residual")


def paradiag_tslab_time(h, cols, c0, bcols):
    _check(load().paradiag_tslab_time(h, _ptr(cols, "cols"), int(c0), int(bcols)), "paradiag_tslab_time")


def paradiag_tslab_update(h, blocks, bcols, U_l, nn):
    _check(load().paradiag_tslab_update(h, _ptr(blocks, "blocks"), int(bcols), _ptr(U_l, "U_l"), int(nn)),
           "paradiag_tslab_update")


def paradiag_destroy(h):
    if h:
        load().paradiag_destroy(h)


class Solver:
    """Owns a handle; shapes follow the C ABI ([nt][ny][nx] iterates, [ny][nx] u0).  With an NCCL id
    the handle is one rank of a sharded problem and every buffer is the rank's row slab
    (self.y0, self.ny rows; see paradiag_init in include/paradiag.h)."""

    def __init__(self, problem, device: int = 0, stream=None, nccl_id: bytes = None, rank: int = 0, nranks: int = 1):
        self.problem = problem if isinstance(problem, pd_problem) else make_problem(problem)
        self.device = device
        self.h = paradiag_init(self.problem, device, stream, nccl_id, rank, nranks)
        n = self.problem.m + 1 if self.problem.bc == 0 else self.problem.m - 1
        self.nx = n
        self.y0, self.ny = paradiag_local_rows(self.h) if self.problem.dim == 2 else (0, 1)
        self.shape = (self.problem.nt, self.ny, self.nx)

    def empty(self):
        import torch
        return torch.empty(self.shape, dtype=torch.float64, device=f"cuda:{self.device}")

    def _full(self, t, name):
        return _check_tensor(t, name, self.shape[0] * self.shape[1] * self.shape[2], self.device)

    def _slice(self, t, name):
        return _check_tensor(t, name, self.shape[1] * self.shape[2], self.device)

    def residual(self, u0, U, r, want_jbar=False):
        return paradiag_residual(self.h, self._slice(u0, "u0"), self._full(U, "U"), self._full(r, "r"), want_jbar)

    def apply_precond(self, r, delta, jbar=0.0):
        paradiag_apply_precond(self.h, self._full(r, "r"), self._full(delta, "delta"), jbar)

    def apply_precond_jt(self, r, delta, jt):
        return paradiag_apply_precond_jt(self.h, self._full(r, "r"), self._full(delta, "delta"), self._slice(jt, "jt"))

    def iterate(self, u0, U, info=None):
        return paradiag_iterate(self.h, self._slice(u0, "u0"), self._full(U, "U"), info)

    def solve(self, u0, U):
        return paradiag_solve(self.h, self._slice(u0, "u0"), self._full(U, "U"))

    def solve_host(self, u0_host):
        uT = np.empty((self.ny, self.nx), dtype=np.float64)
        rc, info = paradiag_solve_host(self.h, np.ascontiguousarray(u0_host, dtype=np.float64).reshape(self.ny, self.nx), uT)
        return uT, rc, info

    def profile(self, enable=True):
        paradiag_profile(self.h, enable)

    def profile_read(self):
        return paradiag_profile_read(self.h)

    def launches_per_iteration(self):
        return paradiag_launches_per_iteration(self.h)

    def close(self):
        if self.h:
            paradiag_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
