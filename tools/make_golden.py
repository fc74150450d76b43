"""Write tests/golden/*_full.json from the ORACLE only (no CUDA path involved).

  python tools/make_golden.py c3 c4 c4e    (c4 / c4e take a few minutes each on 8 cores)

Each file records the oracle's per-window iteration counts, increments, and the iterate at a
fixed set of sample points (drawn from a seeded RNG), plus mass/energy for CH.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import iterate, diagnostics  # noqa: E402
from workloads import config, make_u0  # noqa: E402


def points(p, count, seed):
    rng = np.random.default_rng(seed)
    pts = [(int(rng.integers(p.nt)), int(rng.integers(p.ny)), int(rng.integers(p.nx))) for _ in range(count)]
    return pts + [(p.nt - 1, 0, 0), (p.nt - 1, p.ny - 1, p.nx - 1), (0, p.ny // 2, p.nx // 2)]


def run(name):
    p = config(name)
    u0 = make_u0(p)
    t = time.time()
    hist = []
    out = {"config": name, "source": "oracle/ (tools/make_golden.py)", "windows": []}
    u = u0
    for w in range(p.n_windows):
        h0 = len(hist)
        U, k, conv = iterate.solve_window(p, u, history=hist)
        pts = points(p, 48, 100 + w)
        win = {"iters": k, "converged": bool(conv),
               "rel": [h["rel"] for h in hist[h0:]],
               "points": pts, "values": [float(U[n, iy, ix]) for n, iy, ix in pts],
               "u_max": float(np.abs(U).max())}
        if p.kind.startswith("cahn_hilliard"):
            win["mass_end"] = diagnostics.mass(p, U[-1])
            win["energy_end"] = diagnostics.energy(p, U[-1])
            win["jbar_last"] = hist[-1]["jbar"]
        out["windows"].append(win)
        u = U[-1].copy()
        print(name, "window", w, "iters", k, flush=True)
    if p.kind.startswith("cahn_hilliard"):
        out["mass_u0"] = diagnostics.mass(p, u0)
        out["energy_u0"] = diagnostics.energy(p, u0)
    out["oracle_seconds"] = time.time() - t
    with open(os.path.join(ROOT, "tests", "golden", f"{name}_full.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    for n in sys.argv[1:]:
        run(n)
