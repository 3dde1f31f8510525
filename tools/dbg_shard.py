import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1311_0089_b200 import _native, generators as gen
from paper_1311_0089_b200.grid import GridSpec

a = gen.cfg3_sphere(27)
one = _native.Context(a.spec)
many = _native.Context(a.spec, slabs=[0, 0])
for ctx in (one, many):
    ctx.set_coefficients(a)
u = np.random.default_rng(0).standard_normal((1, 3) + a.spec.shape)
print("apply_system iso diff", np.max(np.abs(one.apply_system(u) - many.apply_system(u))))
E = np.array([[1.0, 0.0, 0.0]])
for mi in (1, 2, 3):
    r1, x1, _ = one.solve_cg(E, 1e-8, mi)
    rP, xP, _ = many.solve_cg(E, 1e-8, mi)
    print(mi, r1[0]["history"], rP[0]["history"], np.max(np.abs(x1 - xP)))
