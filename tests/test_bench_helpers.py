"""bench.py's host-side helpers (CPU): the byte model, the preconditioner summary, the oracle
sample sizing and the reference arm's JSON line shape."""
import json
import os
import subprocess
import sys

import bench
from workloads import config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_precond_summary_uses_the_algorithmic_bytes():
    prof = {"dtt_x_fwd": (2, 20.0), "dtt_y_fwd": (2, 30.0), "time_solve_2d": (2, 26.0), "dtt_y_inv": (2, 30.0),
            "dtt_x_inv": (2, 20.0), "residual": (2, 15.0), "update": (2, 16.0)}
    dofs = 1_000_000
    s = bench.precond_summary(prof, 2, dofs, 6000.0)
    assert abs(s["ms_per_step"] - 63.0) < 1e-12                 # residual / update excluded
    assert s["algorithmic_bytes"] == 80 * dofs                  # 5 passes × 16 B/dof
    assert abs(s["hbm_frac"] - 80 * dofs / 63e-3 / 1e9 / 6000.0) < 1e-12
    assert bench.precond_summary({"residual": (1, 1.0)}, 1, dofs, 6000.0) is None


def test_every_profiled_kernel_has_a_byte_model():
    # the names the library reports (paradiag.cu kKernelNames) that carry HBM traffic
    for k in ("residual", "dtt_x_fwd", "dtt_y_fwd", "time_solve_2d", "dtt_y_inv", "dtt_x_inv", "update",
              "dtt_x_inv_update", "residual_update", "tlong_a_fwd", "tlong_b_fused", "tlong_a_inv",
              "residual_dst_x", "dst_x_inv_update"):
        assert k in bench.BYTES_PER_DOF


def test_oracle_samples_are_bounded():
    assert bench.oracle_sample_problem("c5").m == 64
    c6 = bench.oracle_sample_problem("c6")
    assert c6.nt == 1024 and abs(c6.t_window / c6.nt - config("c6").t_window / config("c6").nt) < 1e-18


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_json_line_is_strict():
    """bench.py prints strict JSON: non-finite floats become null (no NaN / Infinity tokens)."""
    import json
    import bench
    line = {"a": float("nan"), "b": [1.0, float("inf")], "c": {"d": -float("inf"), "e": 2}, "f": "x"}
    out = json.dumps(bench._finite(line), allow_nan=False)
    assert json.loads(out) == {"a": None, "b": [1.0, None], "c": {"d": None, "e": 2}, "f": "x"}
