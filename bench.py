"""Benchmark of the GaNi CG hot path (BASELINE.json metric) on B200.

Headline workload (N = 1): BASELINE configs[3], "cfg4" -- the largest
single-GPU configuration: a 729^3 polycrystal of 512 seeded Voronoi grains
with lognormal SPD tensors (packed, 6 words per voxel), E = (1, 0, 0), CG to
relative residual 1e-8 (132 iterations).  A step is one complete solve; the
metric counts grid points x CG iterations per second.  Synthetic inputs, fp64.
The other BASELINE configurations that fit one GPU are measured in the same
run under ``other_configs``: cfg2 (2187^2, three batched load cases), cfg3
(243^3 sphere, CG) and cfg3's fixed point (A0 = 25.5 I, tol 1e-6).

  value : coefficients resident in HBM before the timed region; solution stays
          on the device.
  e2e   : through the C-ABI binding with HOST buffers: the coefficient field
          uploaded from pinned memory, the solve, the solution downloaded to
          pinned memory, every step.
  roofline: dominant kernel by CUDA-event time; its ALGORITHMIC bytes (SURVEY
          8(d) model) summed over the launches that did work -- the right-hand
          side sweeps (profiled as "<kernel>_rhs"), the first iteration (no
          p_old, no deferred x) and the iterations with fewer active load
          cases are charged what they move -- over its total time, against the
          measured HBM copy bandwidth (MEASURED_PEAKS.json).
  cpu_baseline: the CPU oracle port (numpy pocketfft, the reference's own
          algorithm and calls, single-threaded per process) on the box's host
          cores, one process per core, measured BEFORE any CUDA work.

``--impl reference`` times that CPU implementation alone (the reference arm).
``--gpus N`` (N > 1) without torchrun re-launches itself under
``torch.distributed.run``; cfg3 / cfg4 / cfg5 are then slab-decomposed over the N
ranks (one GPU each, NCCL exchanges inside the library, strong scaling), cfg2
runs independent replicas (weak scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CG operator applications/sec (grid pts×iters/s) and achieved HBM GB/s vs peak"
UNIT = "grid-pt*iter/s"
TOL = 1e-8
MAX_ITER = 2000
W = 8  # bytes per fp64 word


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# --------------------------------------------------------------------------- dist
def relaunch_under_torchrun(n):
    """`bench.py --gpus N` outside torchrun: re-exec as N ranks on this node."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


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

    def __init__(self, name, n=0, world=1):
        from paper_1311_0089_b200 import generators as gen

        self.name = name
        self.method = "cg"
        if name == "cfg2":
            self.n = n or 2187
            self.shape = (self.n, self.n)
            self.loads = np.array(gen.CFG2_LOADS)
            self.nA = 1
            self.desc = (f"cfg2: {self.n}x{self.n} two-phase random medium (contrast 100, seed 2187), "
                         f"3 load cases batched in one CG solve to 1e-8 (BASELINE configs[1])")
        elif name in ("cfg3", "cfg3fp"):
            self.n = n or 243
            self.shape = (self.n,) * 3
            self.loads = np.array([[1.0, 0.0, 0.0]])
            self.nA = 1
            if name == "cfg3":
                self.desc = (f"cfg3: {self.n}^3 centred sphere (radius 0.35 cell, contrast 50), E=(1,0,0), "
                             f"CG to 1e-8 (BASELINE configs[2])")
            else:
                self.method = "fixed_point"
                self.desc = (f"cfg3 fixed point: {self.n}^3 centred sphere (contrast 50), E=(1,0,0), "
                             f"A0 = 25.5 I, update norm to 1e-6 (BASELINE configs[2])")
        elif name == "cfg4":
            self.n = n or 729
            self.shape = (self.n,) * 3
            self.loads = np.array([[1.0, 0.0, 0.0]])
            self.nA = 6
            self.desc = (f"cfg4: {self.n}^3 polycrystal, 512 seeded Voronoi grains (seed 729) with lognormal "
                         f"SPD tensors (packed, 6 words/voxel; held in HBM as 16-bit grain labels + a table of "
                         f"the 512 packed tensors, same values), generated on the device; E=(1,0,0), CG to 1e-8 "
                         f"(BASELINE configs[3])")
        elif name == "cfg5":
            # full size needs >= 2 GPUs of HBM; one GPU runs the 405^3 down-scale
            self.n = n or (1215 if world >= 2 else 405)
            self.shape = (self.n,) * 3
            self.loads = np.array([gen.CFG5_LOAD])
            self.nA = 1
            self.desc = (f"cfg5: {self.n}^3 two-phase medium, seeded overlapping spheres of radius "
                         f"{20.0 * self.n / 1215:g} voxels to 30% volume fraction (contrast 1000), generated on "
                         f"the device; E=(1,1,1)/sqrt3, CG to 1e-8 (BASELINE configs[4]"
                         f"{'' if self.n == 1215 else ', down-scaled from 1215^3'})")
        else:
            raise ValueError(name)
        self.d = len(self.shape)
        self.R = self.loads.shape[0]
        self.N = int(np.prod(self.shape))

    # ---- device setup ------------------------------------------------------
    def host_field(self):
        from paper_1311_0089_b200 import generators as gen

        if self.name == "cfg2":
            return gen.cfg2_random_two_phase(self.n)
        if self.name in ("cfg3", "cfg3fp"):
            return gen.cfg3_sphere(self.n)
        return None

    def setup(self, ctx, host_field=None, count_fn=None, want_labels=False, compress=True):
        """Coefficient field into HBM (upload, or the device generator for cfg4 / cfg5)."""
        from paper_1311_0089_b200 import generators as gen

        if host_field is not None:
            ctx.set_coefficients(host_field)
            self.note_coefficients(ctx)
            return None
        if self.name == "cfg4":
            seeds, packed = gen.cfg4_grains(512, gen.SEEDS["cfg4"], self.n)
            out = ctx.generate_voronoi(seeds, packed, want_labels=want_labels, compress=compress), packed
            self.note_coefficients(ctx)
            return out
        if self.name == "cfg5":
            gen.cfg5_device(ctx, self.n, count_fn=count_fn)
            self.note_coefficients(ctx)
            return None
        ctx.set_coefficients(self.host_field())
        self.note_coefficients(ctx)
        return None

    def note_coefficients(self, ctx):
        """Coefficient words per voxel the first sweep reads from HBM: the packed
        field's nsym, or a 2-byte label when the context holds the phase-indexed form."""
        if getattr(ctx, "n_phases", 0) > 0:
            self.nA = 2.0 / W
        # outer sweep storing F0^-1 q once (plan two_field): one spectrum word per voxel
        # and RHS less written, and one less read by the inverse middle sweep
        self.two_field = bool(ctx.plan_info("two_field")) if hasattr(ctx, "plan_info") else False
        self.fold_fwd = bool(ctx.plan_info("fold_fwd")) if hasattr(ctx, "plan_info") else False
        return self.nA

    # ---- byte model ----------------------------------------------
    def iter_bytes(self):
        """Fixed SURVEY model per CG iteration (B_iter) or fixed-point iteration (B_fp)."""
        c, R, S = self.d, self.R, 2 * self.d - 1
        extra = c * R if self.method == "fixed_point" else 9 * c * R
        return W * self.N * (self.nA + 2 * S * c * R + extra - (2 * R if getattr(self, "two_field", False) else 0)
                                 - (2 * R if getattr(self, "fold_fwd", False) else 0))

    def launch_words(self, kernel, phase, split):
        """(coefficient words read once per launch, words per active RHS) per voxel.

        phase: "rhs" (IN_CONST first sweep / EP_RHS last sweep), "first" (first CG
        iteration: p' = r, no deferred x), "steady", "fp" (fixed-point iteration).
        With ``split`` the packed-coefficient first sweep is a pointwise kernel
        (writes y = A p') followed by the row FFT on y."""
        c, nA = self.d, self.nA
        first_sweep = {"rhs": (nA, c),           # read A ; write spectrum (or y)
                       "first": (nA, 3 * c),     # + read r ; write p'
                       "steady": (nA, 6 * c),    # + read p_old ; x read / write (deferred update)
                       "fp": (nA, 2 * c)}        # read A, e ; write spectrum
        if kernel == "pointwise":
            return first_sweep[phase]
        if kernel == "row_fwd":
            return (0, 2 * c) if split else first_sweep[phase]
        if getattr(self, "fold_fwd", False) and kernel in ("mid_fwd", "outer"):
            # mid_fwd: c fields in, v0 and the folded u = xi1 v1 + xi2 v2 out; outer: 2 in, 2 out
            return (0, 2 * c - 1) if kernel == "mid_fwd" else (0, 2 * c - 2)
        if kernel in ("outer", "mid_inv") and getattr(self, "two_field", False):
            # outer: c fields in, F0^-1 (xi0 q) and t = F0^-1 q out; mid_inv: those two in
            # (t feeds components 1 and 2: ncu sees it come from DRAM once), c fields out
            return (0, 2 * c - 1)
        if kernel in ("mid_fwd", "outer", "mid_inv"):
            return (0, 2 * c)
        if kernel == "row_inv":
            return (0, 2 * c) if phase == "rhs" else (0, 3 * c)  # spectrum in, r / Ap (+ p or e) out
        if kernel == "cg_update":
            return (0, 3 * c)                    # read r, Ap ; write r (x deferred)
        if kernel == "x_flush":
            return (0, 3 * c)                    # read x, p ; write x
        return None

    def kernel_bytes(self, prof, iters, steps, local=1.0):
        """Algorithmic bytes per kernel name over the profiled steps (None: not modelled)."""
        split = "pointwise" in prof
        out = {}
        for name in prof:
            base, _, tag = name.partition("_rhs")
            rhs = name.endswith("_rhs")
            kern = name[:-4] if rhs else name
            if self.launch_words(kern, "steady", split) is None:
                out[name] = None
                continue
            if rhs:
                a, b = self.launch_words(kern, "rhs", split)
                words = a + b * self.R
            elif self.method == "fixed_point":
                a, b = self.launch_words(kern, "fp", split)
                words = sum(a + b * sum(1 for it in iters if it >= i) for i in range(1, max(iters) + 1))
            elif kern == "x_flush":
                words = self.launch_words(kern, "steady", split)[1] * sum(1 for it in iters if it > 0)
            else:
                words = 0
                for i in range(1, max(iters) + 1):
                    act = sum(1 for it in iters if it >= i)
                    a, b = self.launch_words(kern, "first" if i == 1 else "steady", split)
                    # cg_update of the iteration that stops a RHS still runs for it
                    words += a + b * act
            out[name] = W * self.N * local * words * steps
        return out


def config_dict(wl, parallelism):
    return {"workload": wl.desc, "grid": list(wl.shape), "load_cases": wl.R, "tol": TOL,
            "method": wl.method, "parallelism": parallelism,
            "l2": "inputs larger than L2 (per-iteration working set > 126 MB)"}


def copies_table(world, sharded):
    """How many times the phase table goes up per step (once per rank of a sharded run)."""
    return world if sharded else 1


def parallelism_label(world, wl, replicas):
    if world == 1:
        return "single"
    return "replicas" if (wl.d == 2 or replicas) else f"slab{world}"


# --------------------------------------------------------------------------- CPU (oracle port)
_CPU = {}


def _cpu_field(name, n):
    """The workload's coefficient field for the CPU oracle, as full (d, d, *N) tensors.

    cfg4 at 729^3 needs ~170 GB in the reference's layout and ~250 s per iteration
    on one core, so its CPU sample runs the same generator at 243^3 (labels by a
    periodic k-d tree: identical to generators.voronoi_labels up to exact
    distance ties).  cfg5 likewise runs at <= 243^3."""
    from oracle import fftcell_oracle as orc
    from paper_1311_0089_b200 import generators as gen

    if name == "cfg2":
        return orc.isotropic_full(gen.cfg2_random_two_phase(n).components[0], 2), n
    if name in ("cfg3", "cfg3fp"):
        return orc.isotropic_full(gen.cfg3_sphere(n).components[0], 3), n
    if name == "cfg4":
        from scipy.spatial import cKDTree

        n = min(n, 243)
        seeds, packed = gen.cfg4_grains(512, gen.SEEDS["cfg4"], n)
        pts = np.indices((n, n, n)).reshape(3, -1).T.astype(float)
        _, lab = cKDTree(seeds, boxsize=float(n)).query(pts, workers=-1)
        return orc.unpack(np.moveaxis(packed[lab.reshape(n, n, n)], -1, 0), 3), n
    n = min(n, 243)
    return orc.isotropic_full(gen.cfg5_two_phase(n).components[0], 3), n


def _cpu_worker(conn, E, n, d):
    from oracle import fftcell_oracle as orc

    st = orc.CGStepper(_CPU["full"], tuple(E), (n,) * d, (1.0,) * d, TOL)
    t0 = time.perf_counter()
    st.setup()
    conn.send(time.perf_counter() - t0)
    while True:
        k = conn.recv()
        if k is None:
            break
        t0 = time.perf_counter()
        done = 0
        for _ in range(k):
            if not st.step():
                st.setup()  # converged: restart (the sample measures iterations)
            done += 1
        conn.send((done, time.perf_counter() - t0))


class CpuPool:
    """One single-threaded oracle CG per host core (load cases round-robin).  Must
    be created before any CUDA work (the workers are forked)."""

    def __init__(self, wl, procs=None):
        import multiprocessing as mp

        for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[var] = "1"
        self.procs = procs or min(os.cpu_count() or 1, 16)
        full, self.n = _cpu_field(wl.name, wl.n)
        _CPU["full"] = full
        self.N = self.n ** wl.d
        self.wl = wl
        ctx = mp.get_context("fork")
        self.conns, self.ps = [], []
        for w in range(self.procs):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_cpu_worker, args=(b, wl.loads[w % wl.R], self.n, wl.d), daemon=True)
            p.start()
            self.conns.append(a)
            self.ps.append(p)
        _CPU.clear()
        self.setup_s = max(c.recv() for c in self.conns)

    def step(self, k=1):
        """k CG iterations on every worker; returns (grid-pt iterations, seconds)."""
        for c in self.conns:
            c.send(k)
        res = [c.recv() for c in self.conns]
        return self.N * sum(r[0] for r in res), max(r[1] for r in res)

    def close(self):
        for c in self.conns:
            c.send(None)
        for p in self.ps:
            p.join(timeout=30)

    def sample_desc(self, what):
        return (f"{what}; {self.procs} processes (one per host core, single-threaded numpy pocketfft "
                f"restatement of solver.py:142-230), {self.wl.name} generator at {self.n}^{self.wl.d}"
                f"{' (down-scaled: the full size does not fit the reference layout in host RAM)' if self.n != self.wl.n else ''}")


# --------------------------------------------------------------------------- arms
def run_reference(args):
    world, rank, _ = dist_setup()
    wl = Workload(args.config, args.n, world)
    if rank != 0:
        return
    pool = CpuPool(wl)
    work, secs = 0.0, 0.0
    for step in range(args.warmup + args.steps):
        w, s = pool.step(1)
        if step >= args.warmup:
            work += w
            secs += s
    pool.close()
    v = work / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak" if parallelism_label(world, wl, args.replicas) != f"slab{world}"
        else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(wl, parallelism_label(world, wl, args.replicas)),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": pool.procs, "kind": "port",
                         "sample": pool.sample_desc("per step: one CG iteration on every process (setup and "
                                                    "right-hand side untimed)")},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(wl, seconds):
    """Bounded CPU sample for our line: setup, then iterations for ~`seconds`."""
    pool = CpuPool(wl)
    work, secs = 0.0, 0.0
    while secs < seconds:
        w, s = pool.step(1)
        work += w
        secs += s
    pool.close()
    return {"value": work / secs, "unit": UNIT, "cores": pool.procs, "kind": "port",
            "sample": pool.sample_desc(f"{int(work / pool.N / pool.procs)} CG iteration(s) per process after an "
                                       f"untimed setup of {pool.setup_s:.1f} s")}


def roofline_block(wl, prof, iters, steps, ms_prof, peak, peak_kind, local=1.0):
    kb = wl.kernel_bytes(prof, iters, steps, local)
    per_kernel = {}
    for k, (n, ms) in prof.items():
        per_kernel[k] = {"launches": n, "total_ms": ms, "avg_ms": ms / max(n, 1),
                         "GBps": kb[k] / (ms / 1000) / 1e9 if kb.get(k) else None,
                         "bytes": kb.get(k)}
    modelled = {k: v for k, v in prof.items() if kb.get(k)}
    top = max(modelled, key=lambda k: modelled[k][1])
    achieved = kb[top] / (prof[top][1] / 1000) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get(f"{wl.name}/{top}")
    roof = {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic,
            "bytes_per_launch": kb[top] / max(prof[top][0], 1), "avg_launch_ms": prof[top][1] / max(prof[top][0], 1),
            "share_of_step": prof[top][1] / ms_prof,
            "timing": "CUDA events around every launch on the library stream over a second region of the same "
                      "steps; bytes = SURVEY 8(d) model per launch that did work (right-hand side, first and "
                      "steady iterations, active load cases), summed, over the summed launch time"}
    op_names = [k for k in ("pointwise", "row_fwd", "mid_fwd", "outer", "mid_inv", "row_inv") if k in prof]
    op_ms = sum(prof[k][1] for k in op_names)
    op_bytes = sum(kb[k] for k in op_names)
    operator = {"kernels": op_names, "ms_per_iteration": op_ms / steps / max(iters),
                "GBps": op_bytes / (op_ms / 1000) / 1e9}
    operator["frac"] = operator["GBps"] / peak
    return roof, per_kernel, operator


def measure(wl, ctx, args, world, steps, fp_ref=None):
    """Warm-up, timed value region, profiled region.  Returns a dict of results."""
    loads = wl.loads

    if wl.method == "fixed_point":
        scale = np.sqrt(np.sum(loads * loads, axis=1))

        def solve():
            reps, _ = ctx.solve_fixed_point(loads, 1e-6, MAX_ITER, fp_ref, scale, want_x=False)
            return reps
    else:
        def solve():
            reps, _, _ = ctx.solve_cg(loads, TOL, MAX_ITER, want_x=False)
            return reps

    for _ in range(args.warmup):
        reps = solve()
    iters = [r["iterations"] for r in reps]
    launches0 = ctx.launch_count()
    barrier(world)
    ctx.timer_mark(0)
    for _ in range(steps):
        reps = solve()
    ctx.timer_mark(1)
    ms = ctx.timer_elapsed(0, 1)
    launches = ctx.launch_count() - launches0
    assert [r["iterations"] for r in reps] == iters
    psteps = min(steps, args.profile_steps)
    ctx.profile_reset()
    ctx.set_profiling(True)
    barrier(world)
    ctx.timer_mark(4)
    for _ in range(psteps):
        solve()
    ctx.timer_mark(5)
    ms_prof = ctx.timer_elapsed(4, 5)
    ctx.set_profiling(False)
    prof = ctx.profile()
    return {"iters": iters, "ms": max_over_ranks(world, ms), "launches": launches, "prof": prof,
            "psteps": psteps, "ms_prof": ms_prof}


def summarize(wl, res, steps, world, sharded, peak, peak_kind):
    iters = res["iters"]
    copies = 1 if sharded else world
    work_per_step = wl.N * sum(iters)
    value = copies * work_per_step * steps / (res["ms"] / 1000.0)
    local = (wl.shape[0] // world) / wl.shape[0] if sharded else 1.0
    roof, per_kernel, operator = roofline_block(wl, res["prof"], iters, res["psteps"], res["ms_prof"], peak,
                                                peak_kind, local)
    step_ms = res["ms"] / steps
    ib = wl.iter_bytes() * local
    iteration = {"bytes": ib, "ms": step_ms / max(iters), "GBps": ib / (step_ms / max(iters) / 1000) / 1e9}
    iteration["frac"] = iteration["GBps"] / peak
    return value, roof, per_kernel, operator, iteration


def run_gpu(args):
    world, rank, local = dist_setup()
    wl = Workload(args.config, args.n, world)
    label = parallelism_label(world, wl, args.replicas)
    sharded = label.startswith("slab")
    cpu = None
    if world == 1 and not args.no_cpu:  # before any CUDA work (forked workers)
        cpu = cpu_baseline(wl, args.cpu_seconds)

    from paper_1311_0089_b200 import _native
    from paper_1311_0089_b200.grid import GridSpec

    peak, peak_kind = peaks()
    spec = GridSpec((1.0,) * wl.d, wl.shape)
    if sharded:
        from paper_1311_0089_b200 import parallel

        ctx = parallel.distributed_context(spec, device=local)
    else:
        ctx = _native.Context(spec, local)
    count_fn = None
    if sharded and wl.name == "cfg5":
        import torch
        import torch.distributed as dist

        def count_fn(v):
            t = torch.tensor([v], dtype=torch.int64)
            dist.all_reduce(t)
            return int(t.item())
    host = wl.host_field()
    gen_out = wl.setup(ctx, host, count_fn=count_fn, want_labels=(wl.name == "cfg4" and not sharded))

    with ClockSampler(local) as clk:
        res = measure(wl, ctx, args, world, args.steps)
    wl.note_coefficients(ctx)  # the plan is complete once the workspace exists
    value, roof, per_kernel, operator, iteration = summarize(wl, res, args.steps, world, sharded, peak, peak_kind)

    # ---- e2e: host buffers through the C-ABI binding ----------------------------
    import torch
    from types import SimpleNamespace

    R, d = wl.R, wl.d
    x_out = torch.empty((R, d) + wl.shape, dtype=torch.float64, pin_memory=True).numpy()
    field = None
    if host is not None:
        pin = torch.empty(host.components.shape, dtype=torch.float64, pin_memory=True).numpy()
        pin[...] = host.components
        field = SimpleNamespace(isotropic_values=pin[0] if host.isotropic_values is not None else None,
                                components=pin)
    elif wl.name == "cfg4" and gen_out is not None and gen_out[0] is not None and not args.scratch_labels:
        labels, grains = gen_out
        pin = torch.empty((6,) + wl.shape, dtype=torch.float64, pin_memory=True).numpy()
        for m in range(6):
            np.take(grains[:, m], labels, out=pin[m])
        del labels
        field = SimpleNamespace(isotropic_values=None, components=pin)
    if wl.name == "cfg4" and (sharded or args.scratch_labels):
        # the sharded generator keeps no labels: take the whole grid's from a scratch
        # single-device context (every rank for itself), then release it
        from paper_1311_0089_b200 import generators as gen

        scratch = _native.Context(spec, local)
        seeds, grains = gen.cfg4_grains(512, gen.SEEDS["cfg4"], wl.n)
        gen_out = (scratch.generate_voronoi(seeds, grains, want_labels=True, compress=False), grains)
        del scratch
    e2e = None
    e2e_steps = min(args.steps, args.e2e_steps)
    copies = 1 if sharded else world

    def timed_e2e(upload):
        upload()
        ctx.solve_cg(wl.loads, TOL, MAX_ITER, out=x_out)
        barrier(world)
        ctx.timer_mark(2)
        for _ in range(e2e_steps):
            upload()
            ctx.solve_cg(wl.loads, TOL, MAX_ITER, out=x_out)
        ctx.timer_mark(3)
        ms = max_over_ranks(world, ctx.timer_elapsed(2, 3))
        return copies * wl.N * sum(res["iters"]) * e2e_steps / (ms / 1000.0)

    if field is not None:
        h2d = field.components.nbytes if field.isotropic_values is None else field.isotropic_values.nbytes
        h2d += wl.loads.nbytes
        e2e = {"value": timed_e2e(lambda: ctx.set_coefficients(field)), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(x_out.nbytes), "steps": e2e_steps,
               "path": "Context.set_coefficients (pinned host field in the reference's packed layout, deduplicated on "
                       "the device every step) + Context.solve_cg(out=pinned host array)"}
    if wl.name == "cfg4" and gen_out is not None and gen_out[0] is not None and getattr(ctx, "n_phases", 0) > 0:
        # the same step from the phase form a generator or segmentation holds: labels +
        # table go up instead of the expanded field (sharded: the only host form small
        # enough to keep per rank; every rank uploads its own planes)
        lab16 = torch.empty(wl.shape, dtype=torch.uint16, pin_memory=True).numpy()
        lab16[...] = gen_out[0]
        table = np.ascontiguousarray(gen_out[1].T)
        idx = {"value": timed_e2e(lambda: ctx.set_coefficients_indexed(lab16, table)), "unit": UNIT,
               "h2d_bytes_per_step": int(lab16.nbytes + copies_table(world, sharded) * table.nbytes + wl.loads.nbytes),
               "d2h_bytes_per_step": int(x_out.nbytes), "steps": e2e_steps,
               "path": "Context.set_coefficients_indexed (pinned uint16 labels + tensor table) + "
                       "Context.solve_cg(out=pinned host array)"}
        if e2e is None:
            e2e = idx
        else:
            e2e["indexed_upload"] = idx
        del lab16
    if field is not None:
        del field, pin
    del x_out

    exchange = None
    prof = res["prof"]
    if "exchange" in prof:  # spectrum transposes between ranks, broken out
        from paper_1311_0089_b200 import parallel

        cnt, tot = prof["exchange"]
        sent = 16 * sum(int(v) for p, v in enumerate(parallel.exchange_counts(wl.shape, R, world)[rank]) if p != rank)
        exchange = {"per_exchange_ms": tot / cnt, "exchanges_per_iteration": 2,
                    "share_of_step": tot / res["ms_prof"], "bytes_sent_per_gpu": sent,
                    "GBps_per_gpu": sent / (tot / cnt / 1000) / 1e9,
                    "transport": "NCCL send/recv over NVLink (one process per GPU)"}
    del ctx

    # ---- the other single-GPU BASELINE configurations (same run, value only) ------
    others = {}
    if world == 1 and not args.no_others and args.config == "cfg4":
        from paper_1311_0089_b200.material import CoefficientField  # noqa: F401

        for name in ("cfg2", "cfg3", "cfg3fp"):
            ow = Workload(name)
            octx = _native.Context(GridSpec((1.0,) * ow.d, ow.shape), local)
            ow.setup(octx, ow.host_field())
            ores = measure(ow, octx, args, world, args.steps, fp_ref=25.5 * np.eye(3))
            ow.note_coefficients(octx)
            ov, oroof, okern, oop, oit = summarize(ow, ores, args.steps, 1, False, peak, peak_kind)
            others[name] = {"config": config_dict(ow, "single"), "value": ov, "unit": UNIT,
                            "ms_per_step": ores["ms"] / args.steps, "iterations": ores["iters"],
                            "roofline": oroof, "iteration_roofline": oit, "operator_roofline": oop,
                            "kernels": okern}
            del octx

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms"] / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(wl, label),
        "iterations": res["iters"],
        "e2e": e2e,
        "gpu_launches": res["launches"],
        "roofline": roof,
        "iteration_roofline": iteration,
        "operator_roofline": operator,
        "kernels": per_kernel,
        "exchange": exchange,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "other_configs": others or None,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4", choices=["cfg2", "cfg3", "cfg3fp", "cfg4", "cfg5"],
                    help="BASELINE configuration (default cfg4 = configs[3], the largest single-GPU one)")
    ap.add_argument("--n", type=int, default=0, help="override the grid size (0 = BASELINE size)")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--scratch-labels", action="store_true",
                    help="cfg4 on one GPU: take the e2e labels the way a sharded run does (scratch context), for testing")
    ap.add_argument("--no-others", action="store_true", help="skip the other single-GPU configurations")
    ap.add_argument("--profile-steps", type=int, default=3, help="steps of the per-kernel profiled region")
    ap.add_argument("--e2e-steps", type=int, default=5, help="steps of the e2e region (<= --steps)")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas even for 3-D configs")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
