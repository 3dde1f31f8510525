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
    """Max of a per-rank time over the process group (host plumbing over gloo)."""
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
class Workload:
    """One BASELINE configuration: device setup, loads, byte model, CPU sample."""

    def __init__(self, name, n):
        from paper_1311_0089_b200 import generators as gen

        self.name = name
        if name == "cfg2":
            self.n = n or 2187
            self.shape = (self.n, self.n)
            self.loads = np.array(gen.CFG2_LOADS)
            self.nA = 1
            self.desc = (f"cfg2: {self.n}x{self.n} two-phase random medium (contrast 100, seed 2187), "
                         f"3 load cases batched in one CG solve to 1e-8 (BASELINE configs[1])")
        elif name == "cfg3":
            self.n = n or 243
            self.shape = (self.n,) * 3
            self.loads = np.array([[1.0, 0.0, 0.0]])
            self.nA = 1
            self.desc = f"cfg3: {self.n}^3 centred sphere (radius 0.35 cell, contrast 50), E=(1,0,0), CG to 1e-8"
        elif name == "cfg4":
            self.n = n or 729
            self.shape = (self.n,) * 3
            self.loads = np.array([[1.0, 0.0, 0.0]])
            self.nA = 6
            self.desc = (f"cfg4: {self.n}^3 polycrystal, 512 seeded Voronoi grains (seed 729) with lognormal "
                         f"SPD tensors, generated on the device; E=(1,0,0), CG to 1e-8")
        else:
            raise ValueError(name)
        self.d = len(self.shape)
        self.R = self.loads.shape[0]
        self.N = int(np.prod(self.shape))

    def host_field(self):
        from paper_1311_0089_b200 import generators as gen

        if self.name == "cfg2":
            return gen.cfg2_random_two_phase(self.n)
        if self.name == "cfg3":
            return gen.cfg3_sphere(self.n)
        return None

    def setup(self, ctx, host_field=None):
        """Put the coefficient field in HBM (upload, or generate on the device for cfg4)."""
        if self.name == "cfg4":
            from paper_1311_0089_b200 import generators as gen

            seeds, packed = gen.cfg4_grains(512, gen.SEEDS["cfg4"], self.n)
            ctx.generate_voronoi(seeds, packed)
            return 3 * 512 * 8 + 6 * 512 * 8
        ctx.set_coefficients(host_field)
        return host_field.isotropic_values.nbytes

    def iter_bytes(self):
        c, R = self.d, self.R
        S = 2 * self.d - 1
        return 8 * self.N * (self.nA + 2 * S * c * R + 9 * c * R)

    # CG solves defer x += alpha p into the next first sweep (FC_DEFER_X,
    # fc_engine.cu / fc_shard.inc); record_iterates keeps it in cg_update
    defer_x = os.environ.get("FC_DEFER_X", "1") != "0"

    def kernel_bytes(self, name):
        """Algorithmic bytes of one launch (SURVEY 8(d) byte model, CG loop).

        The per-iteration total (iter_bytes) is the fixed SURVEY model; with the
        deferred x update 2cR words move from cg_update to row_fwd and cg_update
        drops its p read, so the per-kernel split follows what each kernel moves."""
        w, c, R, nA = 8, self.d, self.R, self.nA
        dx = 2 * c * R if self.defer_x else 0
        first = w * (nA + 4 * c * R + dx)  # read r, p ; write p' ; write spectrum (+ A ; + x r/w deferred)
        # packed coefficients run the first sweep split (FC_ANISO_SPLIT, default
        # on): a pointwise kernel writes y = A p' (one more field write, which the
        # row FFT reads back) -- charged at the model's bytes plus that round trip
        split = nA > 1 and os.environ.get("FC_ANISO_SPLIT", "1") != "0"
        per = {
            "pointwise": first if split else None,
            "row_fwd": w * 2 * c * R if split else first,
            "mid_fwd": w * 2 * c * R,
            "outer": w * 2 * c * R,
            "mid_inv": w * 2 * c * R,
            "row_inv": w * 3 * c * R,          # read spectrum, write Ap, read p
            "cg_update": w * (3 if self.defer_x else 6) * c * R,  # read r, Ap ; write r (+ read x, p ; write x)
        }.get(name)
        return None if per is None else per * self.N


def _oracle_worker(args):
    name, n, E, seconds = args
    from oracle import fftcell_oracle as orc
    from paper_1311_0089_b200 import generators as gen

    if name == "cfg2":
        a = gen.cfg2_random_two_phase(n)
        full = orc.isotropic_full(a.components[0], 2)
    elif name == "cfg3":
        a = gen.cfg3_sphere(n)
        full = orc.isotropic_full(a.components[0], 3)
    else:
        a = gen.cfg4_polycrystal(n)
        full = orc.unpack(a.components, 3)
    rep = orc.solve_cg(full, tuple(E), a.spec.shape, a.spec.half_periods, TOL, MAX_ITER, max_seconds=seconds)
    return rep["iterations"], rep["loop_seconds"], a.spec.total


def cpu_sample(wl, seconds):
    """Time-bounded oracle CG, one process per load case (the reference is single-threaded).

    cfg4 at 729^3 does not fit the reference's ~440 B/voxel; its sample runs the same
    generator at 81^3 (throughput per grid point is reported)."""
    n = wl.n if wl.name != "cfg4" else min(wl.n, 81)
    with ProcessPoolExecutor(len(wl.loads)) as ex:
        res = list(ex.map(_oracle_worker, [(wl.name, n, E, seconds) for E in wl.loads]))
    work = sum(N * it for it, _, N in res)
    t = max(s for _, s, _ in res)
    its = [it for it, _, _ in res]
    return work, t, its, n


# --------------------------------------------------------------------------- arms
def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    wl = Workload(args.config, args.n)
    total_work, total_t = 0.0, 0.0
    sample = None
    for step in range(args.warmup + args.steps):
        work, t, its, n = cpu_sample(wl, args.cpu_seconds)
        if step >= args.warmup:
            total_work += work
            total_t += t
            sample = (its, n)
    v = total_work / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(wl),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": len(wl.loads), "kind": "port",
                         "sample": f"per step: the first CG iterations of each of the {len(wl.loads)} load case(s) "
                                   f"of {wl.name} at {sample[1]}^{wl.d}, {args.cpu_seconds:g} s each, one process "
                                   f"per load case (numpy pocketfft restatement of solver.py:142-230); "
                                   f"iterations {sample[0]}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(wl, parallelism="replicas"):
    return {"workload": wl.desc, "grid": list(wl.shape), "load_cases": wl.R, "tol": TOL,
            "parallelism": parallelism,
            "l2": "inputs larger than L2 (per-iteration working set > 126 MB)"}


def run_gpu(args):
    world, rank, local = dist_setup()
    from paper_1311_0089_b200 import _native
    from paper_1311_0089_b200.material import CoefficientField
    from paper_1311_0089_b200.grid import GridSpec

    wl = Workload(args.config, args.n)
    loads, R, N, d = wl.loads, wl.R, wl.N, wl.d
    host = wl.host_field()
    spec = GridSpec((1.0,) * d, wl.shape)
    # 3-D configs shard along axis 0 across the ranks (NCCL exchanges inside the
    # library, strong scaling); cfg2 runs independent replicas (weak scaling)
    sharded = world > 1 and d == 3 and not args.replicas
    if sharded:
        from paper_1311_0089_b200 import parallel

        ctx = parallel.distributed_context(spec, device=local)
    else:
        ctx = _native.Context(spec, local)
    wl.setup(ctx, host)

    def solve_resident():
        reps, _, _ = ctx.solve_cg(loads, TOL, MAX_ITER, want_x=False)
        return reps

    for _ in range(args.warmup):
        reps = solve_resident()
    iters = [r["iterations"] for r in reps]
    work_per_step = N * sum(iters)

    # ---- timed: resident inputs (value) --------------------------------------
    # K steps bracketed by stream events, no per-kernel events inside (those
    # cost ~3 % of the step); the per-kernel breakdown comes from a second
    # region of the same K steps with an event pair around every launch.
    launches0 = ctx.launch_count()
    barrier(world)
    with ClockSampler(local) as clk:
        ctx.timer_mark(0)
        for _ in range(args.steps):
            reps = solve_resident()
        ctx.timer_mark(1)
        ms = ctx.timer_elapsed(0, 1)
    launches = ctx.launch_count() - launches0
    assert [r["iterations"] for r in reps] == iters
    ctx.profile_reset()
    ctx.set_profiling(True)
    barrier(world)
    ctx.timer_mark(4)
    for _ in range(args.steps):
        reps = solve_resident()
    ctx.timer_mark(5)
    ms_prof = ctx.timer_elapsed(4, 5)
    ctx.set_profiling(False)
    prof = ctx.profile()
    ms_max = max_over_ranks(world, ms)
    copies = 1 if sharded else world
    value = copies * work_per_step * args.steps / (ms_max / 1000.0)

    # ---- e2e: host buffers through the public API -----------------------------
    import torch

    x_out = torch.empty((R, d) + wl.shape, dtype=torch.float64, pin_memory=True).numpy()
    a_pinned = None
    if host is not None:
        pin_a = torch.empty(host.components.shape, dtype=torch.float64, pin_memory=True).numpy()
        pin_a[...] = host.components
        a_pinned = CoefficientField(host.spec, pin_a)
    h2d = wl.setup(ctx, a_pinned) + loads.nbytes
    ctx.solve_cg(loads, TOL, MAX_ITER, out=x_out)
    d2h = x_out.nbytes
    e2e_steps = max(1, args.steps if wl.name != "cfg4" else 1)
    barrier(world)
    ctx.timer_mark(2)
    for _ in range(e2e_steps):
        wl.setup(ctx, a_pinned)
        ctx.solve_cg(loads, TOL, MAX_ITER, out=x_out)
    ctx.timer_mark(3)
    ms_e2e = max_over_ranks(world, ctx.timer_elapsed(2, 3))
    e2e = copies * work_per_step * e2e_steps / (ms_e2e / 1000.0)

    if rank != 0:
        return
    peak, peak_kind = peaks()
    # sharded: rank 0's kernels process its slab only (planes [0, n0/P))
    local = (wl.shape[0] // world) / wl.shape[0] if sharded else 1.0
    kbytes = wl.kernel_bytes
    wl.kernel_bytes = lambda k: None if kbytes(k) is None else kbytes(k) * local
    kern = {k: v for k, v in prof.items() if wl.kernel_bytes(k) is not None}
    top = max(kern, key=lambda k: kern[k][1])
    avg_ms = kern[top][1] / kern[top][0]
    bytes_launch = wl.kernel_bytes(top)
    achieved = bytes_launch / (avg_ms / 1000.0) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get(f"{wl.name}/{top}")
    step_ms = ms / args.steps
    n_iter = max(iters)
    roofline = {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic,
                "bytes_per_launch": bytes_launch, "avg_launch_ms": avg_ms,
                "share_of_step": kern[top][1] / ms_prof,
                "timing": "CUDA events around every launch on the library stream, over a second region of the "
                          "same K steps (the value region carries no per-kernel events)",
                "profiled_ms_per_step": ms_prof / args.steps}
    per_kernel = {}
    for k, v in prof.items():
        avg = v[1] / max(v[0], 1)
        kb = wl.kernel_bytes(k)
        per_kernel[k] = {"launches": v[0], "avg_ms": avg, "GBps": kb / (avg / 1000) / 1e9 if kb else None}
    ib = wl.iter_bytes() * local  # per GPU
    iteration = {"bytes": ib, "ms": step_ms / n_iter, "GBps": ib / (step_ms / n_iter / 1000) / 1e9}
    iteration["frac"] = iteration["GBps"] / peak
    exchange = None
    if "exchange" in prof:  # spectrum transposes between ranks, broken out
        from paper_1311_0089_b200 import parallel

        cnt, tot = prof["exchange"]
        sent = 16 * sum(int(v) for p, v in enumerate(parallel.exchange_counts(wl.shape, R, world)[rank]) if p != rank)
        exchange = {"per_exchange_ms": tot / cnt, "exchanges_per_iteration": 2,
                    "share_of_step": tot / ms_prof, "bytes_sent_per_gpu": sent,
                    "GBps_per_gpu": sent / (tot / cnt / 1000) / 1e9,
                    "transport": "NCCL send/recv over NVLink (one process per GPU)"}
    op_names = [k for k in ("pointwise", "row_fwd", "mid_fwd", "outer", "mid_inv", "row_inv") if k in prof]
    op_ms = sum(per_kernel[k]["avg_ms"] for k in op_names)
    op_bytes = sum(wl.kernel_bytes(k) for k in op_names)
    operator = {"kernels": op_names, "ms": op_ms, "GBps": op_bytes / (op_ms / 1000) / 1e9}
    operator["frac"] = operator["GBps"] / peak

    cpu = None
    if world == 1 and not args.no_cpu:
        work, t, its, n = cpu_sample(wl, args.cpu_seconds)
        cpu = {"value": work / t, "unit": UNIT, "cores": R, "kind": "port",
               "sample": f"first CG iterations of each of the {R} load case(s) of {wl.name} at {n}^{d}, "
                         f"{args.cpu_seconds:g} s each, one process per load case; iterations {its}"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(wl, f"slab{world}" if sharded else ("replicas" if world > 1 else "single")),
        "iterations": iters,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": launches,
        "roofline": roofline,
        "iteration_roofline": iteration,
        "operator_roofline": operator,
        "kernels": per_kernel,
        "exchange": exchange,
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
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg3", "cfg4"],
                    help="BASELINE configuration (default cfg2 = configs[1], the metric's workload)")
    ap.add_argument("--n", type=int, default=0, help="override the grid size (0 = BASELINE size)")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas even for 3-D configs")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
