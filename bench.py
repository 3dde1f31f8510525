"""Benchmark of the GaNi CG hot path (BASELINE.json metric) on B200.

Workload (BASELINE configs[1], "cfg2"): 2187 x 2187 two-phase random medium
(contrast 100, seed 2187), three load cases E=(1,0),(0,1),(1,1)/sqrt2 batched in
ONE device CG solve to relative residual 1e-8.  A step is one complete batched
solve (about 83 iterations per load case); the metric counts grid points x CG
iterations per second summed over the load cases.  Synthetic inputs, fp64.

  value : coefficients resident in HBM before the timed region; solution stays
          on the device.
  e2e   : the public API with HOST buffers: coefficient upload (pinned), the
          batched solve, solution download (pinned), every step.
  roofline: dominant kernel, algorithmic bytes (SURVEY 8(d) model) per launch /
          its average CUDA-event duration over the timed region vs the measured
          HBM copy bandwidth in MEASURED_PEAKS.json.
  cpu_baseline: the CPU oracle port (numpy pocketfft, the reference's own
          algorithm and calls) on a time-bounded sample, one process per load case.

``--impl reference`` times that CPU implementation alone (the reference arm).
``--gpus N`` under torchrun: independent replicas of the workload, one per GPU
(weak scaling; the slab-decomposed multi-GPU operator is not in this build).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CG operator applications/sec (grid pts×iters/s) and achieved HBM GB/s vs peak"
UNIT = "grid-pt*iter/s"
TOL = 1e-8
MAX_ITER = 2000


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# --------------------------------------------------------------------------- dist
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(world, v):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        rows = [s for s in self.samples if len(s) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        load = [r for r in rows if r[2] not in ("", "0")] or rows
        sm = [float(r[0]) for r in load if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------- workload
def workload(n):
    from paper_1311_0089_b200 import generators as gen

    a = gen.cfg2_random_two_phase(n)
    return a, np.array(gen.CFG2_LOADS)


def kernel_bytes_per_voxel(name, c, R, nA):
    """Algorithmic bytes per voxel of one launch (SURVEY 8(d) byte model, CG loop)."""
    w = 8
    return {
        "row_fwd": w * (nA + 4 * c * R),   # read r, p ; write p' ; write spectrum  (+ A once)
        "mid_fwd": w * 2 * c * R,
        "outer": w * 2 * c * R,
        "mid_inv": w * 2 * c * R,
        "row_inv": w * 3 * c * R,          # read spectrum, write Ap, read p
        "cg_update": w * 6 * c * R,        # read x, r, p, Ap ; write x, r
    }.get(name)


def _oracle_worker(args):
    n, E, seconds = args
    from oracle import fftcell_oracle as orc
    from paper_1311_0089_b200 import generators as gen

    a = gen.cfg2_random_two_phase(n)
    full = orc.isotropic_full(a.components[0], 2)
    rep = orc.solve_cg(full, tuple(E), a.spec.shape, a.spec.half_periods, TOL, MAX_ITER, max_seconds=seconds)
    return rep["iterations"], rep["loop_seconds"]


def cpu_sample(n, loads, seconds):
    """Time-bounded oracle CG, one process per load case (the reference is single-threaded)."""
    with ProcessPoolExecutor(len(loads)) as ex:
        res = list(ex.map(_oracle_worker, [(n, E, seconds) for E in loads]))
    N = n * n
    work = sum(N * it for it, _ in res)
    t = max(s for _, s in res)
    its = [it for it, _ in res]
    return work, t, its


# --------------------------------------------------------------------------- arms
def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    n = args.n
    _, loads = workload(n)
    total_work, total_t = 0.0, 0.0
    sample_its = []
    for step in range(args.warmup + args.steps):
        work, t, its = cpu_sample(n, loads, args.cpu_seconds)
        if step >= args.warmup:
            total_work += work
            total_t += t
            sample_its.append(its)
    v = total_work / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(n),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": len(loads), "kind": "port",
                         "sample": f"per step: the first CG iterations of each of the {len(loads)} load cases "
                                   f"of cfg2 ({n}^2), {args.cpu_seconds:g} s per load case, one process each "
                                   f"(numpy pocketfft restatement of solver.py:142-230); iterations {sample_its[0]}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(n):
    return {"workload": f"cfg2: {n}x{n} two-phase random medium (contrast 100, seed 2187), 3 load cases "
                        f"batched in one CG solve to 1e-8 (BASELINE configs[1])",
            "grid": [n, n], "load_cases": 3, "tol": TOL, "parallelism": "replicas",
            "l2": "inputs larger than L2 (per-iteration working set > 126 MB)"}


def run_gpu(args):
    world, rank, local = dist_setup()
    from paper_1311_0089_b200 import _native
    from paper_1311_0089_b200.material import CoefficientField

    n = args.n
    a_host, loads = workload(n)
    R = len(loads)
    N = n * n
    d = 2
    ctx = _native.Context(a_host.spec, local)
    ctx.set_coefficients(a_host)

    def solve_resident():
        reps, _, _ = ctx.solve_cg(loads, TOL, MAX_ITER, want_x=False)
        return reps

    # warm-up
    for _ in range(args.warmup):
        reps = solve_resident()
    iters = [r["iterations"] for r in reps]
    work_per_step = N * sum(iters)

    # ---- timed: resident inputs (value) --------------------------------------
    ctx.profile_reset()
    ctx.set_profiling(True)
    launches0 = ctx.launch_count()
    barrier(world)
    with ClockSampler(local) as clk:
        ctx.timer_mark(0)
        for _ in range(args.steps):
            reps = solve_resident()
        ctx.timer_mark(1)
        ms = ctx.timer_elapsed(0, 1)
    launches = ctx.launch_count() - launches0
    ctx.set_profiling(False)
    prof = ctx.profile()
    assert [r["iterations"] for r in reps] == iters
    ms_max = max_over_ranks(world, ms)
    value = world * work_per_step * args.steps / (ms_max / 1000.0)

    # ---- e2e: host buffers through the public API -----------------------------
    import torch

    pin_a = torch.empty(a_host.components.shape, dtype=torch.float64, pin_memory=True).numpy()
    pin_a[...] = a_host.components
    a_pinned = CoefficientField(a_host.spec, pin_a)
    x_out = torch.empty((R, d, n, n), dtype=torch.float64, pin_memory=True).numpy()
    h2d = a_pinned.isotropic_values.nbytes + loads.nbytes
    d2h = x_out.nbytes
    for _ in range(1):
        ctx.set_coefficients(a_pinned)
        ctx.solve_cg(loads, TOL, MAX_ITER, out=x_out)
    barrier(world)
    ctx.timer_mark(2)
    for _ in range(args.steps):
        ctx.set_coefficients(a_pinned)
        ctx.solve_cg(loads, TOL, MAX_ITER, out=x_out)
    ctx.timer_mark(3)
    ms_e2e = max_over_ranks(world, ctx.timer_elapsed(2, 3))
    e2e = world * work_per_step * args.steps / (ms_e2e / 1000.0)

    if rank != 0:
        return
    # ---- roofline of the dominant kernel ------------------------------------------
    peak, peak_kind = peaks()
    kern = {k: v for k, v in prof.items() if kernel_bytes_per_voxel(k, d, R, 1) is not None}
    top = max(kern, key=lambda k: kern[k][1])
    nl, avg_ms = kern[top][0], kern[top][1] / kern[top][0]
    bytes_launch = kernel_bytes_per_voxel(top, d, R, 1) * N
    achieved = bytes_launch / (avg_ms / 1000.0) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get(f"cfg2/{top}")
    step_ms = ms / args.steps
    iter_bytes = 728 * N  # B_iter/voxel for cfg2 (R=3, isotropic)
    n_iter_launch = max(iters)
    roofline = {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic,
                "bytes_per_launch": bytes_launch, "avg_launch_ms": avg_ms,
                "share_of_step": kern[top][1] / ms}
    per_kernel = {k: {"launches": v[0], "avg_ms": v[1] / max(v[0], 1),
                      "GBps": (kernel_bytes_per_voxel(k, d, R, 1) * N / (v[1] / max(v[0], 1) / 1000) / 1e9)
                      if kernel_bytes_per_voxel(k, d, R, 1) else None}
                  for k, v in prof.items()}
    iteration = {"bytes": iter_bytes, "ms": step_ms / n_iter_launch,
                 "GBps": iter_bytes / (step_ms / n_iter_launch / 1000) / 1e9}
    iteration["frac"] = iteration["GBps"] / peak

    cpu = None
    if world == 1 and not args.no_cpu:
        work, t, its = cpu_sample(n, loads, args.cpu_seconds)
        cpu = {"value": work / t, "unit": UNIT, "cores": R, "kind": "port",
               "sample": f"first CG iterations of each of the {R} load cases of cfg2 ({n}^2), "
                         f"{args.cpu_seconds:g} s per load case, one process each; iterations {its}"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(n),
        "iterations": iters,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": launches,
        "roofline": roofline,
        "iteration_roofline": iteration,
        "kernels": per_kernel,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=2187, help="grid size (BASELINE cfg2: 2187)")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
