"""Diagnostic: long-window P_α⁻¹ (fused / unfused pass B) vs a numpy-FFT eigenbasis evaluation."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from _helpers import gshape, to_dev, to_host, rel_err
from workloads import twin
from oracle import circulant, spatial
import paper_2304_14021_b200 as pd

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 15
p = twin("c6", nt=nt, t_window=nt / 2.0 ** 20)
r = np.random.default_rng(23).uniform(-1, 1, gshape(p)).reshape(p.nt, p.nx)
g = circulant.gamma(p.nt, p.alpha)
S1 = np.fft.fft(g[:, None] * r, axis=0)
d = circulant.eig_d(p.nt, p.alpha, circulant.inv_dt(p)); e = circulant.eig_e(p.nt, p.alpha, p.theta)
T = spatial.transform_matrix(p.m, p.bc)
mu = spatial.mu(spatial.Lam_grid(p), p).reshape(-1)
S2 = ((S1 @ T.T) / (d[:, None] + e[:, None] * mu[None, :])) @ T.T / (2.0 * p.m)
ref = (np.fft.ifft(S2, axis=0) / g[:, None]).real
for fuse in ("1", "0"):
    os.environ["PARADIAG_TLFUSE"] = fuse
    s = pd.Solver(p)
    dd = s.empty()
    s.apply_precond(to_dev(r.reshape(gshape(p)), p), dd, 0.0)
    out = to_host(dd, p)
    err = np.abs(out - ref)
    i = np.unravel_index(np.argmax(err), err.shape)
    print("fuse", fuse, "rel", rel_err(out, ref), "argmax", i, flush=True)
    s.close()
