"""Golden digest of the UNMODIFIED reference on the cfg5 generator at 405^3.

BASELINE configs[4] (1215^3) does not fit one GPU; its single-GPU stand-in is
the same generator down-scaled to 405^3 (sphere radius 20 x 405 / 1215 voxels,
30% volume fraction, contrast 1000, E = (1,1,1)/sqrt3, CG to 1e-8), the
radix-5 register-FFT length of the cfg5 axis.  Runs the reference's own
``solve_cg`` (one core, ~2-3 h, ~30 GB) in the build container:

    python tests/golden/make_cfg5_405.py

Stored: iterations, residual history, |x|, <A(E + x), E + x> and x at 4096
seeded sample positions (tests/test_gpu_parity.py::test_cfg5_405_full_size).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from fftcell.grid import GridSpec  # noqa: E402
from fftcell.material import CoefficientField, apply_A  # noqa: E402
from fftcell.solver import LoadCase, SolverConfig, solve_cg  # noqa: E402
from fftcell.transforms import GridField, l2_inner, l2_norm  # noqa: E402

from paper_1311_0089_b200 import generators as gen  # noqa: E402

OUT = Path(__file__).resolve().parent
N = 405


def main():
    t0 = time.time()
    ours = gen.cfg5_two_phase(N)
    print(f"generator {time.time() - t0:.1f} s, volume fraction {(ours.components[0] > 1).mean():.5f}", flush=True)
    a = CoefficientField(GridSpec((1.0,) * 3, (N,) * 3), ours.components)
    del ours
    load = LoadCase(gen.CFG5_LOAD)
    t1 = time.perf_counter()
    rep = solve_cg(a, load, SolverConfig(tol=1e-8, max_iter=3000))
    secs = time.perf_counter() - t1
    sol = rep.solution.values
    idx = np.sort(np.random.default_rng(424242).choice(sol.size, size=4096, replace=False))
    tot = GridField(a.spec, sol + load.expand(a.spec).values)
    energy = l2_inner(apply_A(a, tot), tot)
    np.savez_compressed(OUT / "cfg5_405.npz", cg_iterations=rep.iterations, cg_converged=rep.converged,
                        cg_history=np.array(rep.residual_history), cg_message=np.array(rep.message),
                        cg_norm=l2_norm(rep.solution), cg_sample_idx=idx, cg_sample=sol.reshape(-1)[idx],
                        energy=energy, seconds=secs, n=N)
    print(f"cfg5_405: {rep.iterations} iterations, energy {energy!r}, {secs:.0f} s", flush=True)


if __name__ == "__main__":
    main()
