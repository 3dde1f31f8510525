"""Generate golden fixtures by running the UNMODIFIED reference (``fftcell``).

Run in the build container, where ``/root/reference`` exists:

    python tests/golden/make_golden.py small   # seconds; full fields
    python tests/golden/make_golden.py large   # ~40 min on one core; digests

Inputs come from ``paper_1311_0089_b200.generators`` / seeded numpy, so the
GPU tests rebuild the identical arrays on the GPU box (where the reference is
absent) and compare against these files.  Large fields are stored as digests:
iteration counts, residual histories, norms, energies and the values at 4096
seeded sample voxels.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from fftcell import families as rfam  # noqa: E402
from fftcell.analysis import dense_oracle  # noqa: E402
from fftcell.green import ReferenceTensor  # noqa: E402
from fftcell.grid import GridSpec  # noqa: E402
from fftcell.homogenize import effective_tensor  # noqa: E402
from fftcell.material import CoefficientField, apply_A  # noqa: E402
from fftcell.solver import (  # noqa: E402
    LoadCase, SolverConfig, _Projector, apply_system, solve_cg, solve_neumann,
)
from fftcell.transforms import GridField, l2_inner, l2_norm  # noqa: E402

from paper_1311_0089_b200 import generators as gen  # noqa: E402

OUT = Path(__file__).resolve().parent
SAMPLE_SEED = 424242
NSAMPLE = 4096


def ref_field(ours):
    """Rebuild one of our CoefficientFields as the reference's type."""
    spec = GridSpec(ours.spec.half_periods, ours.spec.shape)
    return CoefficientField(spec, ours.components)


def sample_idx(n):
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(n, size=min(NSAMPLE, n), replace=False))


class perturbed_fft:
    """Run the reference with scipy's pocketfft over REVERSED axis order: the same
    mathematics with different rounding.  The difference to the unperturbed run is
    the reference's own reproducibility floor, recorded as ``<prefix>floor``."""

    def __enter__(self):
        import scipy.fft as sf

        self.saved = np.fft.fftn, np.fft.ifftn
        np.fft.fftn = lambda a, axes=None: sf.fftn(a, axes=None if axes is None else axes[::-1])
        np.fft.ifftn = lambda a, axes=None: sf.ifftn(a, axes=None if axes is None else axes[::-1])

    def __exit__(self, *exc):
        np.fft.fftn, np.fft.ifftn = self.saved


def with_floor(prefix, run, full=True):
    """report_dict of run() plus the perturbed-rounding floor (rel. L2 and history)."""
    rep = run()
    out = report_dict(prefix, rep, full)
    with perturbed_fft():
        alt = run()
    ref = rep.solution.values
    nrm = np.linalg.norm(ref)
    out[f"{prefix}floor"] = float(np.linalg.norm(alt.solution.values - ref) / nrm) if nrm > 0 else 0.0
    h, ha = np.array(rep.residual_history), np.array(alt.residual_history)
    m = min(len(h), len(ha))
    out[f"{prefix}floor_hist"] = (float(np.max(np.abs(h[:m] - ha[:m]) / np.maximum(h[:m], h[0])))
                                  if m and h[0] > 0 else 0.0)
    out[f"{prefix}floor_iterations"] = alt.iterations
    return out


def report_dict(prefix, rep, full=True):
    sol = rep.solution.values
    out = {
        f"{prefix}iterations": rep.iterations,
        f"{prefix}converged": rep.converged,
        f"{prefix}history": np.array(rep.residual_history),
        f"{prefix}message": np.array(rep.message),
        f"{prefix}norm": l2_norm(rep.solution),
    }
    if full:
        out[f"{prefix}solution"] = sol
    else:
        idx = sample_idx(sol.size)
        out[f"{prefix}sample_idx"] = idx
        out[f"{prefix}sample"] = sol.reshape(-1)[idx]
    return out


def energy(a, load, rep):
    tot = GridField(a.spec, rep.solution.values + load.expand(a.spec).values)
    return l2_inner(apply_A(a, tot), tot)


def random_spd_packed(shape, rng, shift=0.5):
    d = len(shape)
    B = rng.standard_normal((d, d) + tuple(shape))
    mats = np.einsum("ab...,cb...->ac...", B, B) + shift * np.eye(d).reshape((d, d) + (1,) * d)
    return np.stack([mats[a, b] for a, b in
                     [(a, a) for a in range(d)] + [(a, b) for a in range(d) for b in range(a + 1, d)]])


def save(name, **kw):
    np.savez_compressed(OUT / f"{name}.npz", **kw)
    print(f"wrote {name}.npz", flush=True)


def small():
    # cfg1: 81^2 square inclusion, CG 1e-8, both fixed-point references, A_H.
    a = ref_field(gen.cfg1_square_inclusion())
    load = LoadCase((1.0, 0.0))
    kw = {}
    kw.update(with_floor("cg_", lambda: solve_cg(a, load, SolverConfig(tol=1e-8, max_iter=1000))))
    mean = float(a.components[0].mean())
    kw["fp_mean_lambda"] = mean
    kw.update(with_floor("fpmean_", lambda: solve_neumann(
        a, load, SolverConfig(method="neumann", tol=1e-8, max_iter=1000,
                              reference=ReferenceTensor.scalar(mean, 2)))))
    kw.update(with_floor("fpdef_", lambda: solve_neumann(
        a, load, SolverConfig(method="neumann", tol=1e-8, max_iter=1000))))
    kw["AH"] = effective_tensor(a, SolverConfig(tol=1e-8, max_iter=1000)).matrix
    save("cfg1", **kw)

    # sine1d N=255 (criterion 2): A_H = sqrt(5) +- 1e-6.
    fam = rfam.sine_1d()
    a = fam.sample(fam.default_spec((255,)))
    eff = effective_tensor(a, SolverConfig(tol=1e-10, max_iter=500))
    kw = {"packed": a.components, "AH": eff.matrix}
    kw.update(with_floor("cg_", lambda: solve_cg(a, LoadCase((1.0,)), SolverConfig(tol=1e-10, max_iter=500))))
    kw.update(with_floor("fp_", lambda: solve_neumann(a, LoadCase((1.0,)),
                                                      SolverConfig(method="neumann", tol=1e-8, max_iter=5000))))
    save("sine255", **kw)

    # Checkerboard 27^2 (1, 50): scalar-reference independence.
    a = rfam.checkerboard_2d(1.0, 50.0).sample(GridSpec((1.0, 1.0), (27, 27)))
    kw = {"packed": a.components}
    kw.update(with_floor("none_", lambda: solve_cg(a, LoadCase((1.0, 0.0)), SolverConfig(tol=1e-8, max_iter=500))))
    for lam in (0.5, 10.0):
        kw.update(with_floor(f"lam{lam:g}_", lambda: solve_cg(
            a, LoadCase((1.0, 0.0)),
            SolverConfig(tol=1e-8, max_iter=500, reference=ReferenceTensor.scalar(lam, 2)))))
    save("checker27", **kw)

    # Random SPD fields vs the dense oracle (criterion 3 shapes) + a d=3 one.
    rng = np.random.default_rng(3)
    cases = [((1.0, 1.0), (5, 5), (1.0, 0.5))] * 3 + [((1.0,), (99,), (1.0,))] * 2 + [
        ((1.0, 1.0, 2.0), (3, 3, 3), (1.0, -0.5, 0.25))]
    kw = {"ncase": len(cases)}
    for i, (Y, shape, E) in enumerate(cases):
        spec = GridSpec(Y, shape)
        a = CoefficientField(spec, random_spd_packed(shape, rng))
        kw[f"c{i}_Y"] = np.array(Y)
        kw[f"c{i}_shape"] = np.array(shape)
        kw[f"c{i}_E"] = np.array(E)
        kw[f"c{i}_packed"] = a.components
        kw.update(with_floor(f"c{i}_", lambda: solve_cg(a, LoadCase(E), SolverConfig(tol=1e-13, max_iter=2000))))
        kw[f"c{i}_dense"] = dense_oracle(a, LoadCase(E)).values
    save("dense_small", **kw)

    # Operator / projector outputs on random inputs over many odd shapes.
    rng = np.random.default_rng(11)
    shapes = [((1.0,), (9,)), ((1.0, 1.5), (5, 5)), ((1.0, 1.0, 2.0), (3, 3, 3)),
              ((1.0,), (255,)), ((1.0, 1.0), (45, 45)), ((1.0, 2.0), (15, 33)),
              ((1.0, 0.5, 2.0), (7, 9, 11)), ((1.0, 1.0, 1.0), (15, 15, 15)),
              ((1.3, 1.0, 0.7), (5, 13, 17)), ((1.0, 1.0), (65, 99)), ((1.0,), (133,)),
              ((1.0, 1.0, 1.0), (25, 21, 15)), ((2.0, 1.0), (261, 7))]
    kw = {"ncase": len(shapes)}
    for i, (Y, shape) in enumerate(shapes):
        spec = GridSpec(Y, shape)
        d = len(shape)
        a = CoefficientField(spec, random_spd_packed(shape, rng))
        u = rng.standard_normal((d,) + shape)
        B = rng.standard_normal((d, d))
        A0 = B @ B.T + 0.5 * np.eye(d)
        kw[f"c{i}_Y"] = np.array(Y)
        kw[f"c{i}_shape"] = np.array(shape)
        kw[f"c{i}_packed"] = a.components
        kw[f"c{i}_u"] = u
        kw[f"c{i}_A0"] = A0
        kw[f"c{i}_system"] = apply_system(a, GridField(spec, u)).values
        proj = _Projector(spec, ReferenceTensor(A0))
        kw[f"c{i}_orth"] = proj.apply_orthogonal(u)
        kw[f"c{i}_gamma"] = proj.apply_gamma_ref(u)
        kw[f"c{i}_Au"] = apply_A(a, GridField(spec, u)).values
    save("operators", **kw)

    # cfg3 generator at 27^3: CG 1e-8 (+A_H), fixed point 1e-6 default reference.
    a = ref_field(gen.cfg3_sphere(27))
    kw = {}
    kw.update(with_floor("cg_", lambda: solve_cg(a, LoadCase((1.0, 0.0, 0.0)), SolverConfig(tol=1e-8, max_iter=1000))))
    kw.update(with_floor("fp_", lambda: solve_neumann(a, LoadCase((1.0, 0.0, 0.0)),
                                                      SolverConfig(method="neumann", tol=1e-6, max_iter=5000))))
    kw["AH"] = effective_tensor(a, SolverConfig(tol=1e-8, max_iter=1000)).matrix
    save("sphere27", **kw)

    # cfg4 generator at 27^3 (512 grains, anisotropic packed tensors): CG 1e-8 and A_H.
    seeds, packed = gen.cfg4_grains(512, gen.SEEDS["cfg4"], 27)
    ours = gen.CoefficientField(gen.GridSpec((1.0,) * 3, (27,) * 3),
                                np.moveaxis(packed[gen.voronoi_labels(27, seeds)], -1, 0).copy())
    a = ref_field(ours)
    kw = {"packed": a.components}
    kw.update(with_floor("cg_", lambda: solve_cg(a, LoadCase((1.0, 0.0, 0.0)), SolverConfig(tol=1e-8, max_iter=2000))))
    eff = effective_tensor(a, SolverConfig(tol=1e-8, max_iter=2000))
    kw["AH"] = eff.matrix
    save("poly27", **kw)

    # cfg2 generator at 81^2: three batched loads, CG 1e-8, per-load energies.
    a = ref_field(gen.cfg2_random_two_phase(81))
    kw = {}
    for j, E in enumerate(gen.CFG2_LOADS):
        kw.update(with_floor(f"l{j}_", lambda: solve_cg(a, LoadCase(E), SolverConfig(tol=1e-8, max_iter=2000))))
        rep = solve_cg(a, LoadCase(E), SolverConfig(tol=1e-8, max_iter=2000))
        kw[f"l{j}_energy"] = energy(a, LoadCase(E), rep)
    save("cfg2_81", **kw)

    # Generic-radix 3-D anisotropic grid (primes 5, 7, 11, 13) with non-unit cell.
    rng = np.random.default_rng(5)
    spec = GridSpec((1.0, 1.5, 0.75), (11, 21, 65))
    a = CoefficientField(spec, random_spd_packed(spec.shape, rng))
    kw = {"packed": a.components, "Y": np.array(spec.half_periods), "shape": np.array(spec.shape)}
    kw.update(with_floor("cg_", lambda: solve_cg(a, LoadCase((0.3, -1.0, 0.5)), SolverConfig(tol=1e-9, max_iter=2000))))
    kw.update(with_floor("fp_", lambda: solve_neumann(
        a, LoadCase((0.3, -1.0, 0.5)),
        SolverConfig(method="neumann", tol=1e-7, max_iter=5000,
                     reference=ReferenceTensor(np.diag([3.0, 2.0, 2.5]))))))
    save("generic3d", **kw)


def large():
    t = time.time()
    # cfg2 full size: 2187^2, seed 2187, three loads, CG 1e-8.
    a = ref_field(gen.cfg2_random_two_phase())
    kw = {}
    for j, E in enumerate(gen.CFG2_LOADS):
        t1 = time.perf_counter()
        rep = solve_cg(a, LoadCase(E), SolverConfig(tol=1e-8, max_iter=2000))
        kw[f"l{j}_seconds"] = time.perf_counter() - t1
        kw.update(report_dict(f"l{j}_", rep, full=False))
        kw[f"l{j}_energy"] = energy(a, LoadCase(E), rep)
        print("cfg2 load", j, rep.iterations, kw[f"l{j}_energy"], time.time() - t, flush=True)
    save("cfg2_full", **kw)
    del a

    # cfg4-like and cfg5-like at 81^3.
    seeds, packed = gen.cfg4_grains(512, gen.SEEDS["cfg4"], 81)
    ours = gen.CoefficientField(gen.GridSpec((1.0,) * 3, (81,) * 3),
                                np.moveaxis(packed[gen.voronoi_labels(81, seeds)], -1, 0).copy())
    a = ref_field(ours)
    t1 = time.perf_counter()
    rep = solve_cg(a, LoadCase((1.0, 0.0, 0.0)), SolverConfig(tol=1e-8, max_iter=2000))
    kw = {"seconds": time.perf_counter() - t1, "c_A": a.c_A, "C_A": a.C_A}
    kw.update(report_dict("cg_", rep, full=False))
    kw["energy"] = energy(a, LoadCase((1.0, 0.0, 0.0)), rep)
    save("cfg4_81", **kw)
    print("cfg4_81", rep.iterations, time.time() - t, flush=True)

    ours = gen.cfg5_two_phase(81)
    a = ref_field(ours)
    t1 = time.perf_counter()
    rep = solve_cg(a, LoadCase(gen.CFG5_LOAD), SolverConfig(tol=1e-8, max_iter=3000))
    kw = {"seconds": time.perf_counter() - t1, "volume_fraction": float((ours.components[0] > 1).mean())}
    kw.update(report_dict("cg_", rep, full=False))
    kw["energy"] = energy(a, LoadCase(gen.CFG5_LOAD), rep)
    save("cfg5_81", **kw)
    print("cfg5_81", rep.iterations, time.time() - t, flush=True)

    # cfg3 full size: 243^3 sphere, CG 1e-8 and fixed point 1e-6 (A_ref = 25.5).
    a = ref_field(gen.cfg3_sphere())
    load = LoadCase((1.0, 0.0, 0.0))
    kw = {}
    t1 = time.perf_counter()
    rep = solve_cg(a, load, SolverConfig(tol=1e-8, max_iter=2000))
    kw["cg_seconds"] = time.perf_counter() - t1
    kw.update(report_dict("cg_", rep, full=False))
    kw["cg_energy"] = energy(a, load, rep)
    print("cfg3 cg", rep.iterations, time.time() - t, flush=True)
    save("cfg3_full", **kw)
    t1 = time.perf_counter()
    rep = solve_neumann(a, load, SolverConfig(method="neumann", tol=1e-6, max_iter=2000))
    kw["fp_seconds"] = time.perf_counter() - t1
    kw.update(report_dict("fp_", rep, full=False))
    kw["fp_energy"] = energy(a, load, rep)
    save("cfg3_full", **kw)
    print("cfg3 fp", rep.iterations, time.time() - t, flush=True)


if __name__ == "__main__":
    {"small": small, "large": large}[sys.argv[1]]()
