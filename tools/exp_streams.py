"""Experiment: do independent load cases overlap when run on separate streams?"""
import sys, threading, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1311_0089_b200 import _native, generators as gen

a = gen.cfg2_random_two_phase()
loads = np.array(gen.CFG2_LOADS)
batched = _native.Context(a.spec); batched.set_coefficients(a)
ctxs = [_native.Context(a.spec) for _ in range(3)]
for c in ctxs: c.set_coefficients(a)
for _ in range(2):
    batched.solve_cg(loads, 1e-8, 2000, want_x=False)
    for i, c in enumerate(ctxs): c.solve_cg(loads[i:i+1], 1e-8, 2000, want_x=False)
t0 = time.perf_counter(); reps, _, _ = batched.solve_cg(loads, 1e-8, 2000, want_x=False); t1 = time.perf_counter()
print("batched R=3", t1 - t0, [r["iterations"] for r in reps])
t0 = time.perf_counter()
for i, c in enumerate(ctxs): c.solve_cg(loads[i:i+1], 1e-8, 2000, want_x=False)
t1 = time.perf_counter(); print("serial 3 x R=1", t1 - t0)
out = [None] * 3
def run(i): out[i] = ctxs[i].solve_cg(loads[i:i+1], 1e-8, 2000, want_x=False)[0][0]["iterations"]
th = [threading.Thread(target=run, args=(i,)) for i in range(3)]
t0 = time.perf_counter()
for t in th: t.start()
for t in th: t.join()
t1 = time.perf_counter(); print("concurrent 3 streams", t1 - t0, out)
