import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1311_0089_b200 import _native, generators as gen
os.environ["FC_FUSED_EXCHANGE"] = "0"
a = gen.cfg3_sphere(81)
ctx = _native.Context(a.spec, slabs=[0, 0, 0])
ctx.set_coefficients(a)
ctx.set_profiling(True)
ctx.solve_cg(np.array([[1.0, 0, 0]]), 1e-8, 500, want_x=False)
ctx.set_profiling(False)
print({k: (v[0], round(v[1], 3)) for k, v in ctx.profile().items()})
