"""Per-kernel timing of one operator application (apply_system, all RHS active).

usage: python tools/kbench.py [cfg2|cfg3|cfg4] [n] [reps]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1311_0089_b200 import _native  # noqa: E402
from paper_1311_0089_b200.grid import GridSpec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
nrhs = int(sys.argv[4]) if len(sys.argv) > 4 else 0
wl = bench.Workload(name, n)
if nrhs:
    wl.loads = wl.loads[:nrhs]
    wl.R = nrhs
ctx = _native.Context(GridSpec((1.0,) * wl.d, wl.shape))
wl.setup(ctx, wl.host_field())
u = np.random.default_rng(0).standard_normal((wl.R, wl.d) + wl.shape)
ctx.apply_system(u)
ctx.profile_reset()
ctx.set_profiling(True)
for _ in range(reps):
    ctx.apply_system(u)
ctx.set_profiling(False)
prof = ctx.profile()
print(name, wl.shape, {k: round(ms / cnt, 4) for k, (cnt, ms) in prof.items()})
