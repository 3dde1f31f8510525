"""Small solves covering every default kernel path, for compute-sanitizer:
d=2 rows of 81 (multi-pencil TMA boxes), d=2 rows of 2187 (persistent last
sweep, one-pencil boxes), d=3 81^3 (TMA middle sweep, bulk outer), a packed
anisotropic field (fused packed first sweep) and the fixed point; once with the
default plan and once with the split finalize forced on these small grids."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1311_0089_b200 import CoefficientField, _native  # noqa: E402
from paper_1311_0089_b200.grid import GridSpec  # noqa: E402

rng = np.random.default_rng(1)
for opts, shape in [(o, s) for o in ({}, {"fin_split": 1}) for s in [(81, 81), (9, 2187), (27, 27, 27)]]:
    _native.lib().fc_reset_plan_options()
    for k, v in opts.items():
        _native.lib().fc_set_plan_option(k.encode(), v)
    spec = GridSpec((1.0,) * len(shape), shape)
    d = len(shape)
    a = np.where(rng.random(shape) < 0.4, 10.0, 1.0)
    ctx = _native.Context(spec)
    ctx.set_coefficients(CoefficientField.isotropic(spec, a))
    E = np.eye(d)[:2]
    reps, x, _ = ctx.solve_cg(E, 1e-8, 200)
    ref = np.diag(np.full(d, 5.5))
    fr, _ = ctx.solve_fixed_point(E[:1], 1e-6, 50, ref, [1.0])
    print(opts, shape, [r["iterations"] for r in reps], fr[0]["iterations"], float(np.abs(x).max()))
    # packed symmetric field (split anisotropic first sweep)
    B = rng.standard_normal((d, d) + shape) * 0.3
    mats = np.einsum("ab...,cb...->ac...", B, B) + np.eye(d).reshape((d, d) + (1,) * d)
    pairs = [(i, i) for i in range(d)] + [(i, j) for i in range(d) for j in range(i + 1, d)]
    packed = np.stack([mats[i, j] for i, j in pairs])
    ctx2 = _native.Context(spec)
    ctx2.set_coefficients(CoefficientField(spec, packed))
    reps2, _, _ = ctx2.solve_cg(E, 1e-8, 200)
    print("  aniso", [r["iterations"] for r in reps2])
