"""A/B of plan options (fc_set_plan_option) on full CG solves of a BASELINE config.

usage: python tools/ab_plan.py cfg4 [n] "" "aniso_fused=0" "row_threads=128" ...
Each argument after the size is one variant (comma-separated key=value, "" =
defaults); prints ms per CG iteration and the per-kernel times of one solve.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1311_0089_b200 import _native  # noqa: E402
from paper_1311_0089_b200.grid import GridSpec  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
variants = sys.argv[3:] or [""]
wl = bench.Workload(name, n)
for var in variants:
    opts = dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in var.split(",") if kv)
    compress = bool(opts.pop("compress", 1))  # 0: keep the packed field (no phase index)
    with _native.plan_options(**opts):
        ctx = _native.Context(GridSpec((1.0,) * wl.d, wl.shape))
    wl.setup(ctx, wl.host_field(), compress=compress)
    reps, _, _ = ctx.solve_cg(wl.loads, bench.TOL, bench.MAX_ITER, want_x=False)
    its = max(r["iterations"] for r in reps)
    ctx.timer_mark(0)
    for _ in range(2):
        ctx.solve_cg(wl.loads, bench.TOL, bench.MAX_ITER, want_x=False)
    ctx.timer_mark(1)
    ms = ctx.timer_elapsed(0, 1) / 2
    ctx.profile_reset()
    ctx.set_profiling(True)
    ctx.solve_cg(wl.loads, bench.TOL, bench.MAX_ITER, want_x=False)
    ctx.set_profiling(False)
    prof = ctx.profile()
    ks = " ".join(f"{k}={v[1] / max(v[0], 1):.3f}" for k, v in prof.items() if not k.endswith("_rhs") or k == "row_fwd_rhs")
    print(f"{name} [{var or 'default'}] phases {ctx.n_phases} iterations {its} {ms / its:.4f} ms/iter | {ks}", flush=True)
    del ctx
