#!/usr/bin/env python
"""bench.py — ParaDiag iteration throughput on B200 (BASELINE.json metric).

metric: space-time dof/s per ParaDiag iteration (fp64) and % of HBM roofline.
workload: BASELINE.json configs[4] (c5): 2D linearised Cahn-Hilliard, Neumann, 2049² nodes,
N_t = 512, T = 0.5, α = 1e-4, β = 0.4, ε = 0.01, U⁰ = 0.  A step is one ParaDiag
iteration through the public C ABI (paradiag_iterate): residual + P_α⁻¹ (5 passes) + update and
the 4-scalar read-back.  Inputs (17.2 GB per array) are far larger than L2 (126 MB), so no L2
flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c5]

Multi-GPU (torchrun, N > 1): the c5 grid is sharded in slabs over the ranks (paper_2304_14021_b200/
dist.py) — row slabs for the residual / x transforms / update, column slabs for the y
transforms and the time pass, NCCL all-to-all transposes between them and a 2-row residual halo —
so the total problem is fixed (strong scaling).  --parallelism replicas runs N independent copies
instead (weak scaling).
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_DOF = {  # algorithmic HBM bytes per space-time dof per launch
    "residual": 16.0, "dtt_x_fwd": 16.0, "dtt_y_fwd": 16.0, "time_solve_2d": 16.0,
    "dtt_y_inv": 16.0, "dtt_x_inv": 16.0, "update": 24.0, "dtt_x_inv_update": 24.0,
    "residual_update": 32.0,      # pipelined solve: read U, δ; write U_new, r
    # long windows (k_tlong.cuh): each pass reads and writes one U-sized array (pairs of real
    # pencils packed as one complex pencil: ⌈N_s/2⌉·16 B = N_s·8 B per time row)
    "tlong_a_fwd": 16.0, "tlong_b_fwd": 16.0, "tlong_divide": 16.0, "tlong_b_inv": 16.0, "tlong_a_inv": 16.0,
    "tlong_b_fused": 16.0,        # pass B + divide + pass B⁻¹ (Y read and written once)
    # 1D short rows (k_x1d.cuh): residual fused with the forward x transform (read U, write r̂),
    # inverse x transform fused with the update (read δ̂, U; write U)
    "residual_dst_x": 16.0, "dst_x_inv_update": 24.0,
}


# the kernels of one P_α⁻¹ application (BASELINE.json target: "the preconditioner application at
# ≥ 60% of the B200 HBM roofline"), by engine path
PRECOND_KERNELS = ("dtt_x_fwd", "dtt_y_fwd", "time_solve_2d", "dtt_y_inv", "dtt_x_inv", "dtt_x_inv_update",
                   "time_fwd_1d", "penta_solve", "time_inv_1d", "tlong_a_fwd", "tlong_b_fwd", "tlong_divide",
                   "tlong_b_inv", "tlong_a_inv", "tlong_b_fused")


def precond_summary(prof, steps, dofs, peak):
    """Device time of the P_α⁻¹ kernels per step and the HBM fraction at their algorithmic bytes."""
    ms = sum(tot for k, (n, tot) in prof.items() if k in PRECOND_KERNELS) / max(steps, 1)
    nbytes = sum(BYTES_PER_DOF.get(k, 0.0) * n for k, (n, _) in prof.items() if k in PRECOND_KERNELS) / max(steps, 1) * dofs
    if ms <= 0:
        return None
    return {"ms_per_step": ms, "algorithmic_bytes": nbytes, "achieved_gbs": nbytes / (ms * 1e-3) / 1e9,
            "hbm_frac": nbytes / (ms * 1e-3) / 1e9 / peak,
            "kernels": [k for k in prof if k in PRECOND_KERNELS]}


def ncu_counters(name):
    """DRAM bytes per launch and FP64-pipe utilisation of kernel `name` from the committed ncu
    --set full capture of the c5 bench (profiles/ncu_counters.json, tools/ncu_counters.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_counters.json")) as f:
            d = json.load(f)
        k = d["kernels"].get(name) or {}
        return {"traffic": k.get("traffic"), "fp64_pipe_pct": k.get("fp64_pipe_pct"),
                "source": "profiles/ncu_counters.json <- " + d.get("source", "?")}
    except Exception:
        return {}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
            "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
            "clocks_event_reasons.sw_power_cap"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for r in self.samples if len(r) >= 7 and r[0].isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [int(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


def oracle_sample_problem(name):
    """Bounded sample of the workload for the CPU oracle: same physics and N_t, 65² nodes (2D);
    1D long windows (c6): same h and Δt, N_t = 1024 (the naive O(N_t²) DFT bounds the sample)."""
    from workloads import twin, config
    p = config(name)
    if p.dim == 1 and p.nt > 4096:
        return twin(name, nt=1024, t_window=p.t_window * 1024 / p.nt)
    return twin(name, m=64)


def time_oracle(name, steps, warmup):
    """Time the oracle (as it stands) on the bounded sample; returns (dof/s, cores, desc, s/step)."""
    import numpy as np
    from oracle import iterate
    from workloads import make_u0
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] or [os.cpu_count()])
    except Exception:
        cores = os.cpu_count()
    p = oracle_sample_problem(name)
    u0 = make_u0(p)
    if p.dim == 1:
        u0 = u0.reshape(-1)            # the oracle's 1D layout
    U = iterate.initial_iterate(p, u0)
    for _ in range(warmup):
        U, _ = iterate.iterate_once(p, u0, U)
    ts = []
    for _ in range(max(steps, 1)):
        t0 = time.perf_counter()
        U, _ = iterate.iterate_once(p, u0, U)
        ts.append(time.perf_counter() - t0)
    dt = statistics.median(ts)
    desc = (f"oracle iterate_once (numpy fp64, naive O(N_t^2) DFT, dense DCT-I matmuls) on a "
            f"{p.ny}x{p.nx} x N_t={p.nt} twin of {name} ({p.dofs} dofs), median of {len(ts)} iteration(s) "
            f"after {warmup} warm-up" + ("; 1D: banded LU + refinement per bin" if p.dim == 1 else ""))
    return p.dofs / dt, cores, desc, dt


class EventTimer:
    """Device time of code regions (collectives) on the launching stream, summed per name."""

    def __init__(self, stream):
        import torch
        self.torch, self.stream, self.pending, self.tot, self.cnt = torch, stream, [], {}, {}

    def __call__(self, name):
        timer = self

        class _Ctx:
            def __enter__(self_):
                self_.e0 = timer.torch.cuda.Event(enable_timing=True)
                self_.e1 = timer.torch.cuda.Event(enable_timing=True)
                self_.e0.record(timer.stream)

            def __exit__(self_, *a):
                self_.e1.record(timer.stream)
                timer.pending.append((name, self_.e0, self_.e1))
                return False
        return _Ctx()

    def collect(self):
        self.torch.cuda.synchronize()
        for name, e0, e1 in self.pending:
            self.tot[name] = self.tot.get(name, 0.0) + e0.elapsed_time(e1)
            self.cnt[name] = self.cnt.get(name, 0) + 1
        self.pending = []
        return {k: self.tot[k] / self.cnt[k] for k in self.tot}


def run_sharded(args, p, rank, world, local, dev, stream, u0, cfg, metric):
    """c5 (or any 2D linear config) sharded over the ranks by the LIBRARY (include/paradiag.h
    paradiag_init with an NCCL id, csrc/shard.cu): rank 0 draws the NCCL id, torch.distributed
    broadcasts it, every rank's handle owns its communicator and runs the halo exchange, the two
    all-to-all transposes and the stop-rule all-reduce itself (strong scaling: the whole problem is
    fixed, value = total dofs / max-rank time)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2304_14021_b200 as pd
    from dataclasses import replace as _replace
    obj = [pd.paradiag_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    nid = obj[0]
    pk = _replace(p, fixed_iters=args.steps)
    s = pd.Solver(pk, device=local, stream=stream.cuda_stream, nccl_id=nid, rank=rank, nranks=world)
    y0, nyl = s.y0, s.ny
    u0_l = torch.from_numpy(np.ascontiguousarray(u0[y0:y0 + nyl])).to(dev)
    U_l = s.empty()
    info = None
    for _ in range(args.warmup):
        info = s.iterate(u0_l, U_l, info)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        ev0.record(stream)
        rc, sinfo = s.solve(u0_l, U_l)          # exactly K iterations (host loop, NCCL inside)
        ev1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms = ev0.elapsed_time(ev1)
    # per-kernel split: a second, profiled run of the same K iterations
    s.profile(True)
    s.solve(u0_l, U_l)
    torch.cuda.synchronize()
    prof = s.profile_read()
    s.profile(False)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps
    value = p.dofs / (ms_step * 1e-3)
    local_dofs = p.nt * nyl * p.n
    peak, peak_src = measured_peaks()
    kernels = {}
    for name, (n, tot) in prof.items():
        avg = tot / max(n, 1)
        bpd = BYTES_PER_DOF.get(name)
        kernels[name] = {"avg_ms": avg, "gbs": (bpd * local_dofs / (avg * 1e-3) / 1e9) if bpd else None}
    top = max(prof.items(), key=lambda kv: kv[1][1]) if prof else None
    roof = None
    if top:
        name, (n, tot) = top
        avg = tot / n
        bpd = BYTES_PER_DOF.get(name, 16.0)
        ach = bpd * local_dofs / (avg * 1e-3) / 1e9
        roof = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "peak_source": peak_src, "traffic": None, "algorithmic_bytes_per_launch": bpd * local_dofs,
                "per": "rank 0 (its row / column slab)"}
    # NVLink: the bytes one transpose sends per rank (the (row slab r) x (column slab q) blocks of
    # the peers), timed as a standalone NCCL all-to-all of that size after the timed region
    from paper_2304_14021_b200.dist import split
    rows = split(p.n, world)
    sent_elems = p.nt * nyl * (p.n - rows[rank][1])
    nvlink = None
    if world > 1:
        send = torch.empty(sent_elems + world, dtype=torch.float64, device=dev)
        recv = torch.empty_like(send)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        dist.barrier()
        e0.record(stream)
        for _ in range(reps):
            dist.all_to_all_single(recv, send)
        e1.record(stream)
        torch.cuda.synchronize()
        tt = torch.tensor([e0.elapsed_time(e1) / reps], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        a2a_ms = float(tt.item())
        nb = 8 * send.numel() * (world - 1) / world
        nvlink = {"achieved": nb / (a2a_ms * 1e-3) / 1e9, "peak": 770.0, "unit": "GB/s",
                  "frac": nb / (a2a_ms * 1e-3) / 1e9 / 770.0, "peak_source": "guide: measured peer copy per direction",
                  "bytes_per_alltoall": nb, "alltoall_ms": a2a_ms,
                  "measured": "standalone NCCL all-to-all of one transpose's byte count (max over ranks)"}
    e2e = None
    if not args.no_e2e:                      # H2D u0 rows, K = 3 iterations, D2H u_Nt rows
        obj = [pd.paradiag_nccl_unique_id() if rank == 0 else None]     # one id per communicator
        dist.broadcast_object_list(obj, src=0)
        se = pd.Solver(_replace(p, fixed_iters=p.fixed_iters or 3), device=local, stream=stream.cuda_stream,
                       nccl_id=obj[0], rank=rank, nranks=world)
        K = p.fixed_iters or 3
        u0h = torch.from_numpy(np.ascontiguousarray(u0[y0:y0 + nyl])).pin_memory()
        outh = torch.empty((nyl, p.n), dtype=torch.float64).pin_memory()
        Ue = se.empty()
        dist.barrier()
        t0 = time.perf_counter()
        u0d = u0h.to(dev, non_blocking=True)
        se.solve(u0d, Ue)
        outh.copy_(Ue[-1], non_blocking=True)
        torch.cuda.synchronize()
        tt = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te = float(tt.item())
        e2e = {"value": K * p.dofs / te, "unit": "dof/s", "h2d_bytes_per_step": int(p.ns * 8),
               "d2h_bytes_per_step": int(p.ns * 8), "step": f"H2D u0 slabs, {K} sharded iterations, D2H u_Nt slabs",
               "seconds_per_step": te}
        se.close()
    launches = sum(n for n, _ in prof.values())
    if rank == 0:
        line = {"metric": metric, "value": value, "unit": "dof/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(cfg, parallelism=f"slab{world}: library-owned NCCL communicator (paradiag_init with an "
                                                 f"NCCL id): row slabs (residual, x transforms, update) / column "
                                                 f"slabs (y transforms, time pass), two all-to-alls + a 2-row halo "
                                                 f"per iteration, max all-reduce of the stop rule",
                               step="one iteration of a K-iteration sharded paradiag_solve (host loop)"),
                "roofline": roof, "nvlink": nvlink, "cpu_baseline": None, "e2e": e2e,
                "gpu_launches": launches * world, "clocks": clk.summary(), "kernels": kernels,
                "precond": precond_summary(prof, args.steps, local_dofs, peak),
                "last_iter": {"last_rel": float(sinfo.last_rel[0])}}
        print(json.dumps(_finite(line), allow_nan=False), flush=True)
    s.close()
    dist.destroy_process_group()
    return 0


def run_tslab(args, p, rank, world, local, dev, stream, u0, cfg, metric):
    """c6 (1D long window) sharded over the ranks in time slabs (dist.TimeSlabRank): contiguous time
    rows for the residual / x transforms / update, x-mode column blocks of all N_t rows for the
    four-step time pass, two NCCL all-to-alls per iteration (strong scaling: the whole window is
    fixed; value = total dofs / max-rank time)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2304_14021_b200 as pd
    from paper_2304_14021_b200 import dist as pdist
    ops = pdist.TslabOps(p, local, stream.cuda_stream)
    rk = pdist.TimeSlabRank(ops, rank, world)
    comm = pdist.TorchComm()
    nn, nx = rk.nn, rk.nx
    u0_d = torch.from_numpy(np.ascontiguousarray(u0).reshape(-1)).to(dev)

    def fresh_U():
        if p.init == "zero":
            return torch.zeros(nn * nx, dtype=torch.float64, device=dev)
        return u0_d.reshape(1, nx).expand(nn, nx).contiguous().reshape(-1)

    U_l = fresh_U()
    for _ in range(args.warmup):
        rk.iterate(u0_d, U_l, comm)
    timer = EventTimer(stream)
    pd.paradiag_profile(ops.h, True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            dmax, umax = rk.iterate(u0_d, U_l, comm, timer)
        ev1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms = ev0.elapsed_time(ev1)
    prof = pd.paradiag_profile_read(ops.h)
    pd.paradiag_profile(ops.h, False)
    coll = timer.collect()
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    value = p.dofs / (ms_step * 1e-3)
    local_dofs = nn * nx
    peak, peak_src = measured_peaks()
    kernels = {}
    for name, (n, tot) in prof.items():
        avg = tot / max(n, 1)
        bpd = BYTES_PER_DOF.get(name)
        kernels[name] = {"avg_ms": avg, "share": tot / (ms if ms > 0 else 1),
                         "gbs": (bpd * local_dofs / (avg * 1e-3) / 1e9) if bpd else None}
    roof = None
    if prof:
        name, (n, tot) = max(prof.items(), key=lambda kv: kv[1][1])
        avg = tot / n
        bpd = BYTES_PER_DOF.get(name, 16.0)
        ach = bpd * local_dofs / (avg * 1e-3) / 1e9
        roof = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "peak_source": peak_src, "traffic": None, "algorithmic_bytes_per_launch": bpd * local_dofs,
                "per": "rank 0 (its time rows / x-mode block)"}
    sent = 8 * nn * rk.bc * (world - 1)           # bytes this rank sends per all-to-all
    nvlink = None
    if world > 1:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        dist.barrier()
        e0.record(stream)
        for _ in range(reps):
            comm.all_to_all(rk.cols, rk.blocks, rk.splits, rk.splits)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        a2a_ms = float(t.item())
        nvlink = {"achieved": sent / (a2a_ms * 1e-3) / 1e9, "peak": 770.0, "unit": "GB/s",
                  "frac": sent / (a2a_ms * 1e-3) / 1e9 / 770.0, "peak_source": "guide: measured peer copy per direction",
                  "bytes_per_alltoall": sent, "alltoall_ms": a2a_ms,
                  "measured": "standalone forward all-to-all of the iteration's blocks (max over ranks)",
                  "in_iteration_ms": {k: coll[k] for k in coll}}
    e2e = None
    if not args.no_e2e:
        K = p.fixed_iters or 3
        u0h = torch.from_numpy(np.ascontiguousarray(u0).reshape(-1)).pin_memory()
        outh = torch.empty(nx, dtype=torch.float64).pin_memory()
        dist.barrier()
        t0 = time.perf_counter()
        u0e = u0h.to(dev, non_blocking=True)
        Ue = fresh_U()
        for _ in range(K):
            rk.iterate(u0e, Ue, comm)
        outh.copy_(Ue[(nn - 1) * nx:], non_blocking=True)
        torch.cuda.synchronize()
        tt = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te = float(tt.item())
        e2e = {"value": K * p.dofs / te, "unit": "dof/s", "h2d_bytes_per_step": int(nx * 8),
               "d2h_bytes_per_step": int(nx * 8), "step": f"H2D u0, {K} time-slab iterations, D2H u_Nt (last rank)",
               "seconds_per_step": te}
    launches = sum(n for n, _ in prof.values()) + args.steps          # + the stats reset per step
    if rank == 0:
        line = {"metric": metric, "value": value, "unit": "dof/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(cfg, parallelism=f"tslab{world}: time rows {nn} per rank (residual, x transforms, "
                                                 f"update) / x-mode blocks of {rk.bc} (four-step time pass), two NCCL "
                                                 f"all-to-alls + one halo row per iteration"),
                "roofline": roof, "nvlink": nvlink, "cpu_baseline": None, "e2e": e2e,
                "gpu_launches": launches * world, "clocks": clk.summary(), "kernels": kernels,
                "last_iter": {"delta_max": dmax, "u_max": umax}}
        print(json.dumps(_finite(line), allow_nan=False), flush=True)
    ops.close()
    dist.destroy_process_group()
    return 0


def _finite(obj):
    """The JSON line with non-finite floats as null (strict JSON: no NaN / Infinity tokens)."""
    if isinstance(obj, float):
        return obj if math.isfinite(obj) else None
    if isinstance(obj, dict):
        return {k: _finite(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_finite(v) for v in obj]
    return obj


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="per-kernel event timing (on by default)")
    ap.add_argument("--mode", default="solve", choices=["solve", "iterate"],
                    help="time one K-iteration paradiag_solve (pipelined engine) or K paradiag_iterate calls")
    ap.add_argument("--parallelism", default="auto", choices=["auto", "slab", "tslab", "replicas"],
                    help="N > 1: slab-sharded (strong scaling, default for 2D linear configs), time slabs "
                         "(strong scaling, default for the 1D long window c6) or replicas")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from workloads import config, make_u0
    p = config(args.config)
    metric = "space-time dof/s per ParaDiag iteration (fp64)"
    desc = {
        "c1": f"BASELINE.json configs[0] (c1): 1D biharmonic, u = u_xx = 0, {p.nx} interior points, N_t={p.nt}, "
              f"T={p.t_window}, alpha={p.alpha}, u0 = sin(pi x)",
        "c2": f"BASELINE.json configs[1] (c2): 1D linearised Cahn-Hilliard, Neumann, {p.nx} nodes, N_t={p.nt}, "
              f"T={p.t_window}, alpha={p.alpha}, beta={p.beta}, eps={p.eps}",
        "c3": f"BASELINE.json configs[2] (c3): 2D biharmonic, u = Lap u = 0, {p.ny}x{p.nx} interior (512x512 grid), "
              f"N_t={p.nt}, T={p.t_window}, alpha={p.alpha}",
        "c4": f"BASELINE.json configs[3] (c4): 2D Cahn-Hilliard PinT-I, Neumann, {p.ny}x{p.nx} nodes, N_t={p.nt} per "
              f"window, dt={p.t_window / p.nt}, alpha={p.alpha}, eps={p.eps}; timed on window 1 (damped "
              f"averaged-Jacobian iteration)",
        "c5": f"BASELINE.json configs[4] (c5): 2D linearised Cahn-Hilliard, Neumann, {p.ny}x{p.nx} nodes, N_t={p.nt}, "
              f"T={p.t_window}, alpha={p.alpha}, beta={p.beta}, eps={p.eps}, U0=0",
        "c6": f"c6 (SURVEY §8(f) NEXT-3, P:692-699): 1D biharmonic, u = u_xx = 0, h = 1/{p.m} ({p.nx} unknowns), "
              f"N_t={p.nt} (2^20 power-of-two form), T={p.t_window}, alpha={p.alpha}",
        "c6n": f"c6n (SURVEY §8(f) NEXT-3 as the paper states it, P:692-699): 1D biharmonic, Neumann (P:84-87), "
               f"h = 1/{p.m} ({p.nx} nodes), N_t={p.nt} = 2^6 5^6 (dt = 1e-6, mixed-radix time pass), T={p.t_window}, "
               f"alpha={p.alpha}",
    }
    cfg = {"workload": desc.get(args.config, args.config),
           "dofs_per_iteration": p.dofs,
           "l2": (f"inputs {p.dofs * 8 / 1e9:.3g} GB/array >> 126 MB L2 (no flush needed)" if p.dofs * 8 > 4 * 126e6
                  else "arrays fit in L2: warm-L2 numbers")}

    if args.impl == "reference":
        if rank != 0:
            return 0
        v, cores, desc, dt = time_oracle(args.config, args.steps, args.warmup)
        line = {"metric": metric, "value": v, "unit": "dof/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference", "config": cfg,
                "cpu_baseline": {"value": v, "unit": "dof/s", "cores": cores, "kind": "oracle", "sample": desc},
                "e2e": {"value": v, "unit": "dof/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(_finite(line), allow_nan=False), flush=True)
        return 0

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2304_14021_b200 as pd

    torch.cuda.set_device(local)
    # exactly what the library's sharded entry points accept (paradiag_init_slab / tslab_check)
    slab_ok = p.dim == 2 and p.kind in ("biharmonic", "linear_ch") and p.theta == 1.0 and \
        64 <= p.m <= 2048 and 32 <= p.nt <= 1024
    tslab_ok = p.dim == 1 and p.kind in ("biharmonic", "linear_ch") and p.nt > 4096 and \
        (p.nx <= 64 or (p.bc == "neumann" and p.nx == 65))
    if args.parallelism == "slab" and not slab_ok:
        raise SystemExit(f"--parallelism slab: {args.config} is not shardable in slabs "
                         "(2D linear kinds, theta = 1, 64 <= m <= 2048, 32 <= N_t <= 1024)")
    if args.parallelism == "tslab" and not tslab_ok:
        raise SystemExit(f"--parallelism tslab: {args.config} is not a 1D long window (N_t > 4096, N_x <= 64)")
    sharded = slab_ok and (args.parallelism == "slab" or (world > 1 and args.parallelism == "auto"))
    tslab = tslab_ok and (args.parallelism == "tslab" or (world > 1 and args.parallelism == "auto"))
    if world > 1 or sharded or tslab:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    u0 = make_u0(p)
    if sharded:
        return run_sharded(args, p, rank, world, local, dev, stream, u0, cfg, metric)
    if tslab:
        return run_tslab(args, p, rank, world, local, dev, stream, u0, cfg, metric)
    u0_d = torch.from_numpy(u0).to(dev)
    s = pd.Solver(p, device=local, stream=stream.cuda_stream)
    U = torch.zeros(s.shape, dtype=torch.float64, device=dev)       # U⁰ = 0 (R#5)
    info = pd.pd_iter_info()
    # mode "solve" (default): the K timed steps are one paradiag_solve of exactly K iterations (the
    # pipelined engine: each iteration's update rides in the next residual); mode
    # "iterate": K calls of paradiag_iterate (residual, P_α⁻¹, separate update)
    from dataclasses import replace as _replace
    if args.mode == "solve":                # exactly K iterations of one window (windows are sequential)
        s.close()
        s = pd.Solver(_replace(p, fixed_iters=args.steps, n_windows=1), device=local, stream=stream.cuda_stream)
    for _ in range(args.warmup):            # W untimed iterations on the timed handle
        info = s.iterate(u0_d, U, info)
    if args.mode == "solve":
        s.solve(u0_d, U)                    # untimed: captures the device-side loop (CUDA graph) once
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # timed region: no per-kernel events (profiling would force the host loop), the graph loop runs
    with Clocks(local) as clk:
        ev0.record(stream)
        if args.mode == "solve":
            rc, sinfo = s.solve(u0_d, U)
        else:
            for _ in range(args.steps):
                info = s.iterate(u0_d, U, info)
        ev1.record(stream)
        torch.cuda.synchronize()
    if args.mode == "solve":
        info.delta_max = float("nan")
        info.u_max = float(U.abs().max())
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    # per-kernel split: a SECOND run of the same K iterations with CUDA events around every kernel
    # (host loop, one stream sync per iteration); its own wall time is reported beside it
    s.profile(True)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    if args.mode == "solve":
        s.solve(u0_d, U)
    else:
        for _ in range(args.steps):
            s.iterate(u0_d, U, info)
    pe1.record(stream)
    torch.cuda.synchronize()
    prof_ms = pe0.elapsed_time(pe1)
    prof = s.profile_read()
    s.profile(False)
    # kernels of the timed region: the profiled run launched the same iteration kernels; the graph
    # adds one stop-rule kernel (k_loop_decide) per iteration
    launches = (sum(n for n, _ in prof.values()) + args.steps if args.mode == "solve"
                else args.steps * s.launches_per_iteration())
    s.close()                               # free its buffers before the e2e handle allocates
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = world * p.dofs / (ms_step * 1e-3)

    # roofline of the dominant kernel (largest device time in the timed region)
    peak, peak_src = measured_peaks()
    top = max(prof.items(), key=lambda kv: kv[1][1]) if prof else None
    roof = None
    kernels = {}
    for name, (n, tot) in prof.items():
        avg = tot / max(n, 1)
        bpd = BYTES_PER_DOF.get(name)
        kernels[name] = {"avg_ms": avg, "share": tot / (prof_ms if prof_ms > 0 else 1),
                         "gbs": (bpd * p.dofs / (avg * 1e-3) / 1e9) if bpd else None}
    if top:
        name, (n, tot) = top
        avg = tot / n
        bpd = BYTES_PER_DOF.get(name, 16.0)
        ach = bpd * p.dofs / (avg * 1e-3) / 1e9
        nc = ncu_counters(name) if args.config == "c5" else {}
        roof = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "peak_source": peak_src, "traffic": nc.get("traffic"),
                "algorithmic_bytes_per_launch": bpd * p.dofs,
                # the secondary bound: FP64-pipe utilisation of the same kernel
                "fp64_pipe_pct": nc.get("fp64_pipe_pct"),
                "counters_source": nc.get("source")}
    # whole-iteration HBM efficiency at the design byte count: the algorithmic bytes
    # of the kernels that ran, per step
    design_bytes = sum(BYTES_PER_DOF.get(k, 0.0) * n for k, (n, _) in prof.items()) / args.steps * p.dofs

    # end-to-end through the host-buffer C-ABI call (H2D u0, K iterations, D2H u_{N_t})
    e2e = None
    if not args.no_e2e:
        from dataclasses import replace
        pe = replace(p, fixed_iters=p.fixed_iters or 3)
        se = pd.Solver(pe, device=local, stream=stream.cuda_stream)
        u0h = np.ascontiguousarray(u0)
        se.solve_host(u0h)           # warm-up (allocates the library-owned iterate)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        reps = 2
        t0 = time.perf_counter()
        for _ in range(reps):
            uT, rc, sinfo = se.solve_host(u0h)
        te = (time.perf_counter() - t0) / reps
        if world > 1:
            t = torch.tensor([te], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": world * pe.fixed_iters * pe.n_windows * pe.dofs / te, "unit": "dof/s",
               "h2d_bytes_per_step": int(u0h.nbytes), "d2h_bytes_per_step": int(uT.nbytes + 32 * pe.fixed_iters),
               "step": f"paradiag_solve_host: H2D u0, {pe.n_windows} window(s) x {pe.fixed_iters} iterations, D2H u_Nt",
               "seconds_per_step": te}
        se.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, desc, dt = time_oracle(args.config, 3, 1)
        cpu = {"value": v, "unit": "dof/s", "cores": cores, "kind": "oracle", "sample": desc}

    if rank == 0:
        line = {"metric": metric, "value": value, "unit": "dof/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(cfg, parallelism="replicas" if world > 1 else "single-gpu",
                               step=("one iteration of a K-iteration paradiag_solve (device-side loop: CUDA "
                                     "graph with a conditional node; residual, P_alpha^-1, update); per-kernel "
                                     "times from a second, event-profiled run of the same K iterations"
                                     if args.mode == "solve" else "one paradiag_iterate")),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches,
                "clocks": clk.summary(), "kernels": kernels,
                "profiled_run_ms_per_step": prof_ms / args.steps,
                "iteration_hbm_frac_at_design_bytes": design_bytes / (ms_step * 1e-3) / 1e9 / peak,
                "precond": precond_summary(prof, args.steps, p.dofs, peak),
                "last_iter": {"delta_max": (None if args.mode == "solve" else info.delta_max),   # solve: per-window
                              "u_max": info.u_max,                                               # data only
                              "last_rel": (float(sinfo.last_rel[0]) if args.mode == "solve" else None)}}
        print(json.dumps(_finite(line), allow_nan=False), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
