"""Per-iteration time of the slab-decomposed CG with P slabs emulated on one
GPU: fused exchange vs copy-engine exchange vs a single slab.

usage: python tools/shard_bench.py [n] [P ...]
"""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1311_0089_b200 import _native, generators as gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 243
Ps = [int(p) for p in sys.argv[2:]] or [2, 4]
a = gen.cfg3_sphere(n)
E = np.array([[1.0, 0.0, 0.0]])


def run(slabs, fused=True):
    os.environ["FC_FUSED_EXCHANGE"] = "1" if fused else "0"
    ctx = _native.Context(a.spec, slabs=slabs) if slabs else _native.Context(a.spec)
    ctx.set_coefficients(a)
    ctx.solve_cg(E, 1e-8, 2000, want_x=False)
    t0 = time.perf_counter()
    reps, _, _ = ctx.solve_cg(E, 1e-8, 2000, want_x=False)
    dt = time.perf_counter() - t0
    return reps[0]["iterations"], 1000 * dt / reps[0]["iterations"]


it, ms = run(None)
print(f"n={n} single slab: {it} iterations, {ms:.3f} ms/iter")
for P in Ps:
    for fused in (True, False):
        it, ms = run([0] * P, fused)
        print(f"  P={P} ({'fused' if fused else 'copy'} exchange): {it} iterations, {ms:.3f} ms/iter")
