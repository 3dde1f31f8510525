"""cfg3 (243^3 sphere, contrast 50) Moulinec-Suquet fixed point to 1e-6 with the
default reference A0 = (1 + 50)/2 I (BASELINE configs[2]): iterations, time per
iteration, byte-model roofline (B_fp = B_op + w N R c)."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1311_0089_b200 import _native, generators as gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 243
a = gen.cfg3_sphere(n)
ctx = _native.Context(a.spec)
ctx.set_coefficients(a)
E = np.array([[1.0, 0.0, 0.0]])
ref = 25.5 * np.eye(3)
ctx.solve_fixed_point(E, 1e-6, 5000, ref, [1.0], want_x=False)
ctx.timer_mark(0)
reps, _ = ctx.solve_fixed_point(E, 1e-6, 5000, ref, [1.0], want_x=False)
ctx.timer_mark(1)
ms = ctx.timer_elapsed(0, 1)
it = reps[0]["iterations"]
N = n ** 3
d, R, nA, S = 3, 1, 1, 5
b_it = 8 * N * (nA + 2 * S * d * R + d * R)
peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
print(json.dumps({"config": f"cfg3 fixed point {n}^3", "iterations": it, "converged": reps[0]["converged"],
                  "ms_per_iteration": ms / it, "grid_pt_iter_per_s": N * it / (ms / 1000),
                  "GBps": b_it / (ms / it / 1000) / 1e9, "frac": b_it / (ms / it / 1000) / 1e9 / peak}))
