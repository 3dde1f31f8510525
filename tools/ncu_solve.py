"""Driver for ncu captures: one CG solve of a BASELINE config, bounded iterations.

usage: python tools/ncu_solve.py cfg4 [max_iter] [n] [plan options: key=value,...]
e.g. ncu --set full -k regex:"k_(row|mid|outer|cg)" -s 12 -c 6 -o out python tools/ncu_solve.py cfg4 4
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1311_0089_b200 import _native  # noqa: E402
from paper_1311_0089_b200.grid import GridSpec  # noqa: E402

name = sys.argv[1]
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n = int(sys.argv[3]) if len(sys.argv) > 3 else 0
opts = dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in (sys.argv[4] if len(sys.argv) > 4 else "").split(",") if kv)
wl = bench.Workload(name, n)
with _native.plan_options(**opts):
    ctx = _native.Context(GridSpec((1.0,) * wl.d, wl.shape))
wl.setup(ctx, wl.host_field())
reps, _, _ = ctx.solve_cg(wl.loads, bench.TOL, max_iter, want_x=False)
print(name, [r["iterations"] for r in reps])
