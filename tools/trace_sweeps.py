"""Per-CTA phase timelines of the sweeps (experimental FC_TRACE build).

usage: tools/exp_build.sh trace -DFC_TRACE=1 && FC_LIB=exp/trace.so python tools/trace_outer.py [cfg2|cfg4]
Stamps (globaltimer, thread 0 of the first 8192 CTAs of each kernel):
0 CTA start, 1 input staged, 2 forward / first transform(s) done, 3 compute done,
4 store issued, 5 store source drained.
"""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1311_0089_b200 import _native  # noqa: E402
from paper_1311_0089_b200.grid import GridSpec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
wl = bench.Workload(name, 0)
ctx = _native.Context(GridSpec((1.0,) * wl.d, wl.shape))
wl.setup(ctx, wl.host_field())
reps, _, _ = ctx.solve_cg(wl.loads, bench.TOL, 3, want_x=False)
n = 6 * 8 * 8192
buf = (ctypes.c_ulonglong * n)()
lib = ctypes.CDLL(str(_native.LIB_PATH))
lib.fc_debug_trace(buf, n)
T = np.frombuffer(buf, dtype=np.uint64).reshape(6, 8192, 8).astype(np.int64)
names = ["outer (d=2)", "row_fwd_pk", "mid_fwd", "outer_seq", "mid_inv", "row_inv"]
ph = ["stage_in", "transform_1", "rest_compute", "issue_store", "store_drain"]
for kid in range(6):
    t = T[kid]
    t = t[(t[:, 0] > 0) & (t[:, 5] > 0)]
    if len(t) == 0:
        continue
    t = t[1000:] if len(t) > 4000 else t  # steady state
    d = np.diff(t[:, :6], axis=1)
    life = (t[:, 5] - t[:, 0]).mean() / 1e3
    print(f"{names[kid]}: {len(t)} CTAs, lifetime mean {life:.2f} us")
    for k, nm in enumerate(ph):
        print(f"   {nm:14s} mean {d[:, k].mean() / 1e3:7.2f} us  p10 {np.percentile(d[:, k], 10) / 1e3:7.2f}  p90 {np.percentile(d[:, k], 90) / 1e3:7.2f}")
