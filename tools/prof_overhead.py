"""cfg2 batched CG solve timed with and without per-kernel event profiling."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1311_0089_b200 import _native  # noqa: E402
from paper_1311_0089_b200.grid import GridSpec  # noqa: E402

wl = bench.Workload("cfg2", 0)
ctx = _native.Context(GridSpec((1.0,) * wl.d, wl.shape))
wl.setup(ctx, wl.host_field())
for _ in range(2):
    ctx.solve_cg(wl.loads, 1e-8, 2000, want_x=False)
for prof in (False, True, False, True):
    ctx.set_profiling(prof)
    ctx.timer_mark(0)
    for _ in range(3):
        reps, _, _ = ctx.solve_cg(wl.loads, 1e-8, 2000, want_x=False)
    ctx.timer_mark(1)
    ctx.set_profiling(False)
    it = max(r["iterations"] for r in reps)
    print("profiling", prof, "ms/iter %.4f" % (ctx.timer_elapsed(0, 1) / 3 / it))
