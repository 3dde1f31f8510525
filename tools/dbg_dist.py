import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch  # noqa
from paper_1311_0089_b200 import _native, generators as gen
a = gen.cfg3_sphere(27)
dist = _native.Context.distributed(a.spec, 1, 0, 0, _native.nccl_unique_id())
dist.set_coefficients(a)
u = np.random.default_rng(0).standard_normal((1, 3) + a.spec.shape)
print("apply_system", np.abs(dist.apply_system(u)).max(), flush=True)
r, x, _ = dist.solve_cg(np.array([[1.0, 0, 0]]), 1e-8, 500)
print(r[0]["iterations"])
