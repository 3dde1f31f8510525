"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden fixtures and the CPU oracle on the same seeded inputs.

Gates (BASELINE north_star): solution within 1e-9 relative L2, A_H within
1e-10 relative, CG / fixed-point iteration counts identical, identical
fixed-point divergence reports.  Operator outputs are checked at 1e-12
(tolerances.PROJECTOR of the reference, tolerances.py:13)."""

import numpy as np
import pytest

from conftest import (
    curl_residual, golden, log_parity, mean_residual, random_gradient_field, random_spd_packed, rel_l2,
)
from oracle import fftcell_oracle as orc
from paper_1311_0089_b200 import (
    CoefficientField, ConvergenceError, GridField, GridSpec, LoadCase, ReferenceTensor, SolverConfig,
    apply_A, apply_system, effective_tensor, generators as gen, residual_norm, solve, solve_batch, solve_cg,
    solve_neumann,
)
from paper_1311_0089_b200.solver import _Projector

pytestmark = pytest.mark.gpu

SOL_TOL = 1e-9
AH_TOL = 1e-10


def field(Y, shape, packed):
    return CoefficientField(GridSpec(tuple(Y), tuple(int(s) for s in shape)), packed)


def _floor(g, key):
    return float(g[key]) if key in g.files else 0.0


def check_report(rep, g, prefix, case=None):
    """Iterations, converged flag and message identical; residual history and
    solution within max(gate, 10 x the reference's own rounding floor).  The floor
    is the difference between two runs of the unmodified reference that differ
    only in FFT rounding (tests/golden/make_golden.py::perturbed_fft)."""
    ref_it = int(g[f"{prefix}iterations"])
    hist = np.array(rep.residual_history)
    ref_hist = g[f"{prefix}history"]
    sol_tol = max(SOL_TOL, 10 * _floor(g, f"{prefix}floor"))
    hist_tol = max(1e-9, 10 * _floor(g, f"{prefix}floor_hist"))
    rec = {"case": case or prefix, "iterations": rep.iterations, "ref_iterations": ref_it,
           "floor": _floor(g, f"{prefix}floor"), "sol_tol": sol_tol}
    if f"{prefix}solution" in g:
        ref = g[f"{prefix}solution"]
        if np.linalg.norm(ref) == 0:
            rec["sol_err"] = float(np.max(np.abs(rep.solution.values)))
            rec["exact_zero"] = True
        else:
            rec["sol_err"] = rel_l2(rep.solution.values, ref)
    else:
        idx = g[f"{prefix}sample_idx"]
        got = rep.solution.values.reshape(-1)[idx]
        # relative L2 over the sampled voxels themselves (not against the full-field norm)
        rec["sol_err"] = rel_l2(got, g[f"{prefix}sample"])
    m = min(len(hist), len(ref_hist))
    if m and ref_hist[0] > 0:  # relative to max(entry, first entry): CG decays, divergent FP grows
        rec["hist_dev"] = float(np.max(np.abs(hist[:m] - ref_hist[:m]) / np.maximum(ref_hist[:m], ref_hist[0])))
    else:
        rec["hist_dev"] = 0.0
    if len(ref_hist) > 1 and "cg" in str(rep.method):
        # stopping margin of the last non-final iterate: ratio / tol
        rec["last_ratio"] = float(ref_hist[-2] / ref_hist[0]) if len(ref_hist) > 1 else None
    log_parity(rec)
    assert rep.iterations == ref_it, (prefix, rep.iterations, ref_it)
    assert rep.converged == bool(g[f"{prefix}converged"])
    assert rep.message == str(g[f"{prefix}message"])
    assert hist.shape == ref_hist.shape
    assert rec["hist_dev"] <= hist_tol, rec
    if rec.get("exact_zero"):
        assert rec["sol_err"] == 0.0
    else:
        assert rec["sol_err"] <= sol_tol, rec


# ---- operators --------------------------------------------------------------

def test_operators_match_reference_on_odd_grids():
    g = golden("operators")
    for i in range(int(g["ncase"])):
        a = field(g[f"c{i}_Y"], g[f"c{i}_shape"], g[f"c{i}_packed"])
        u = GridField(a.spec, g[f"c{i}_u"])
        scale = max(1.0, float(np.max(np.abs(u.values))))
        np.testing.assert_allclose(apply_A(a, u).values, g[f"c{i}_Au"], rtol=0, atol=1e-14 * scale * a.C_A)
        np.testing.assert_allclose(apply_system(a, u).values, g[f"c{i}_system"], rtol=0,
                                   atol=1e-12 * scale * a.C_A)
        proj = _Projector(a.spec, ReferenceTensor(g[f"c{i}_A0"]))
        np.testing.assert_allclose(proj.apply_orthogonal(u.values), g[f"c{i}_orth"], rtol=0, atol=1e-12 * scale)
        np.testing.assert_allclose(proj.apply_gamma_ref(u.values), g[f"c{i}_gamma"], rtol=0,
                                   atol=1e-12 * scale * np.max(np.abs(g[f"c{i}_gamma"])) / max(
                                       1e-300, np.max(np.abs(g[f"c{i}_gamma"]))) + 1e-12 * scale)


def test_constant_fields_give_exact_zero_projection():
    for shape in [(81, 81), (9, 9), (27, 27, 27), (15, 21), (7, 11, 13), (255,)]:
        spec = GridSpec((1.0,) * len(shape), shape)
        proj = _Projector(spec)
        u = np.broadcast_to(np.arange(1, len(shape) + 1, dtype=float).reshape((-1,) + (1,) * len(shape)),
                            (len(shape),) + shape).copy()
        assert np.max(np.abs(proj.apply_orthogonal(u))) == 0.0, shape


def test_projection_identities(rng):
    for shape, Y in [((5, 5), (1.0, 1.5)), ((3, 3, 3), (1.0, 1.0, 2.0)), ((9,), (1.0,)), ((33, 65), (1.0, 1.0))]:
        spec = GridSpec(Y, shape)
        proj = _Projector(spec)
        u = rng.standard_normal((len(shape),) + shape)
        once = proj.apply_orthogonal(u)
        twice = proj.apply_orthogonal(once)
        assert np.max(np.abs(twice - once)) <= 1e-12 * max(1.0, np.max(np.abs(u)))
        assert curl_residual(once, Y) <= 1e-12
        assert mean_residual(once) <= 1e-12


def test_apply_system_symmetric_on_subspace(rng):
    shape, Y = (5, 5), (1.0, 1.0)
    a = CoefficientField(GridSpec(Y, shape), random_spd_packed(shape, rng))
    u = GridField(a.spec, random_gradient_field(shape, Y, rng))
    v = GridField(a.spec, random_gradient_field(shape, Y, rng))
    lhs = np.sum(apply_system(a, u).values * v.values)
    rhs = np.sum(u.values * apply_system(a, v).values)
    assert lhs == pytest.approx(rhs, rel=1e-11, abs=1e-11)


# ---- solvers vs reference goldens ---------------------------------------------

def test_cfg1_cg_fixed_point_and_effective_tensor():
    g = golden("cfg1")
    a = gen.cfg1_square_inclusion()
    load = LoadCase((1.0, 0.0))
    check_report(solve_cg(a, load, SolverConfig(tol=1e-8, max_iter=1000)), g, "cg_")
    lam = float(g["fp_mean_lambda"])
    rep = solve_neumann(a, load, SolverConfig(method="fixed_point", tol=1e-8, max_iter=1000,
                                              reference=ReferenceTensor.scalar(lam, 2)))
    check_report(rep, g, "fpmean_")
    assert "divergent" in rep.message and rep.iterations == 18
    check_report(solve_neumann(a, load, SolverConfig(method="neumann", tol=1e-8, max_iter=1000)), g, "fpdef_")
    eff = effective_tensor(a, SolverConfig(tol=1e-8, max_iter=1000))
    np.testing.assert_allclose(eff.matrix, g["AH"], rtol=AH_TOL, atol=AH_TOL * np.max(np.abs(g["AH"])))


def test_sine1d_harmonic_mean():
    g = golden("sine255")
    a = field((1.0,), (255,), g["packed"])
    eff = effective_tensor(a, SolverConfig(tol=1e-10, max_iter=500))
    check_report(eff.per_case_reports[0], g, "cg_")
    assert abs(eff.matrix[0, 0] - float(g["AH"][0, 0])) <= AH_TOL * abs(float(g["AH"][0, 0]))
    assert abs(eff.matrix[0, 0] - np.sqrt(5.0)) <= 1e-6
    check_report(solve_neumann(a, LoadCase((1.0,)), SolverConfig(method="neumann", tol=1e-8, max_iter=5000)),
                 g, "fp_")


def test_scalar_reference_independence():
    g = golden("checker27")
    a = field((1.0, 1.0), (27, 27), g["packed"])
    load = LoadCase((1.0, 0.0))
    check_report(solve_cg(a, load, SolverConfig(tol=1e-8, max_iter=500)), g, "none_")
    for lam in (0.5, 10.0):
        cfg = SolverConfig(tol=1e-8, max_iter=500, reference=ReferenceTensor.scalar(lam, 2))
        check_report(solve_cg(a, load, cfg), g, f"lam{lam:g}_")


def test_dense_oracle_equivalence():
    g = golden("dense_small")
    for i in range(int(g["ncase"])):
        a = field(g[f"c{i}_Y"], g[f"c{i}_shape"], g[f"c{i}_packed"])
        rep = solve_cg(a, LoadCase(tuple(g[f"c{i}_E"])), SolverConfig(tol=1e-13, max_iter=2000))
        # tol = 1e-13 sits at the rounding floor: the reference test (test_solver.py:125-133,
        # test_acceptance.py:63-80) gates convergence and the dense solution, not the count
        assert rep.converged and abs(rep.iterations - int(g[f"c{i}_iterations"])) <= 2
        dev = float(np.max(np.abs(rep.solution.values - g[f"c{i}_dense"])))
        log_parity({"case": f"dense_small/c{i}", "dense_dev": dev, "iterations": rep.iterations,
                    "ref_iterations": int(g[f"c{i}_iterations"])})
        assert dev <= 1e-10


@pytest.mark.parametrize("name", ["sphere27", "poly27"])
def test_3d_cg_and_effective_tensor(name):
    g = golden(name)
    a = gen.cfg3_sphere(27) if name == "sphere27" else field((1.0,) * 3, (27,) * 3, g["packed"])
    check_report(solve_cg(a, LoadCase((1.0, 0.0, 0.0)), SolverConfig(tol=1e-8, max_iter=2000)), g, "cg_")
    eff = effective_tensor(a, SolverConfig(tol=1e-8, max_iter=2000))
    np.testing.assert_allclose(eff.matrix, g["AH"], rtol=0, atol=AH_TOL * np.max(np.abs(g["AH"])))
    if name == "sphere27":
        check_report(solve_neumann(a, LoadCase((1.0, 0.0, 0.0)),
                                   SolverConfig(method="neumann", tol=1e-6, max_iter=5000)), g, "fp_")


def test_cfg2_generator_batched_loads():
    g = golden("cfg2_81")
    a = gen.cfg2_random_two_phase(81)
    reps = solve_batch(a, [LoadCase(E) for E in gen.CFG2_LOADS], SolverConfig(tol=1e-8, max_iter=2000))
    E = np.array(gen.CFG2_LOADS)
    en = a.device().energy(E, np.stack([r.solution.values for r in reps]))
    for j, rep in enumerate(reps):
        check_report(rep, g, f"l{j}_")
        assert abs(en[j, j] - float(g[f"l{j}_energy"])) <= AH_TOL * abs(float(g[f"l{j}_energy"]))


def test_generic_radix_anisotropic_3d():
    g = golden("generic3d")
    a = field(g["Y"], g["shape"], g["packed"])
    load = LoadCase((0.3, -1.0, 0.5))
    check_report(solve_cg(a, load, SolverConfig(tol=1e-9, max_iter=2000)), g, "cg_")
    ref = ReferenceTensor(np.diag([3.0, 2.0, 2.5]))
    check_report(solve_neumann(a, load, SolverConfig(method="neumann", tol=1e-7, max_iter=5000, reference=ref)),
                 g, "fp_")


# ---- behaviour the reference tests pin ------------------------------------------

def test_homogeneous_medium_is_exact():
    spec = GridSpec((1.0, 1.0), (81, 81))
    a = CoefficientField.isotropic(spec, np.full(spec.shape, 3.5))
    load = LoadCase((1.2, -0.7))
    rep = solve_cg(a, load, SolverConfig(tol=1e-10))
    assert rep.iterations == 0 and rep.converged
    assert np.max(np.abs(rep.solution.values)) == 0.0
    assert residual_norm(a, load, rep.solution) <= 1e-12
    eff = effective_tensor(a, SolverConfig(tol=1e-10))
    assert np.array_equal(eff.matrix, 3.5 * np.eye(2))


def test_fixed_point_matching_reference_converges_immediately():
    spec = GridSpec((1.0, 1.0), (9, 9))
    a = CoefficientField.isotropic(spec, np.full(spec.shape, 2.0))
    rep = solve_neumann(a, LoadCase((1.0, 0.0)),
                        SolverConfig(method="neumann", tol=1e-10, reference=ReferenceTensor.scalar(2.0, 2)))
    assert rep.converged and rep.iterations == 1
    assert np.max(np.abs(rep.solution.values)) <= 1e-12


def test_max_iter_exhaustion_and_warm_start():
    g = golden("sine255")
    a = CoefficientField(GridSpec((1.0,), (255,)), g["packed"])
    load = LoadCase((1.0,))
    rep = solve_cg(a, load, SolverConfig(tol=1e-12, max_iter=2))
    assert not rep.converged and rep.iterations == 2 and rep.message == ""
    cfg = SolverConfig(tol=1e-8, max_iter=500)
    cold = solve_cg(a, load, cfg)
    warm = solve(a, load, cfg, init=cold.solution)
    assert warm.converged and warm.iterations <= 2
    assert np.allclose(warm.solution.values, cold.solution.values, atol=1e-8)
    full = orc.unpack(g["packed"], 1)
    ref = orc.solve_cg(full, (1.0,), (255,), (1.0,), 1e-8, 500, init=cold.solution.values)
    assert warm.iterations == ref["iterations"]


def test_record_iterates_stay_in_subspace():
    g = golden("sine255")
    a = CoefficientField(GridSpec((1.0,), (255,)), g["packed"])
    rep = solve_cg(a, LoadCase((1.0,)), SolverConfig(tol=1e-10, max_iter=500), record_iterates=True)
    assert len(rep.iterates) == rep.iterations + 1
    for it in rep.iterates:
        assert mean_residual(it.values) <= 1e-10
        assert curl_residual(it.values, (1.0,)) <= 1e-10


def test_effective_tensor_non_convergence_raises():
    g = golden("sine255")
    a = CoefficientField(GridSpec((1.0,), (255,)), g["packed"])
    with pytest.raises(ConvergenceError) as exc:
        effective_tensor(a, SolverConfig(tol=1e-12, max_iter=1))
    assert len(exc.value.reports) == 1 and not exc.value.reports[-1].converged


def test_random_fields_vs_oracle(rng):
    """Seeded random SPD fields on assorted odd 2-D/3-D grids, CG and fixed point."""
    cases = [((1.0, 1.0), (45, 63), (1.0, 0.5)), ((1.0, 2.0, 0.5), (9, 15, 25), (0.2, 1.0, -0.4)),
             ((1.0, 1.0, 1.0), (21, 9, 35), (1.0, 0.0, 0.0))]
    for Y, shape, E in cases:
        packed = random_spd_packed(shape, rng)
        a = CoefficientField(GridSpec(Y, shape), packed)
        full = orc.unpack(packed, len(shape))
        rep = solve_cg(a, LoadCase(E), SolverConfig(tol=1e-9, max_iter=3000))
        ref = orc.solve_cg(full, E, shape, Y, 1e-9, 3000)
        assert rep.iterations == ref["iterations"]
        assert rel_l2(rep.solution.values, ref["solution"]) <= SOL_TOL
        lam = 0.5 * (a.c_A + a.C_A)
        rep = solve_neumann(a, LoadCase(E), SolverConfig(method="neumann", tol=1e-6, max_iter=3000))
        ref = orc.solve_neumann(full, E, shape, Y, 1e-6, 3000, lam * np.eye(len(shape)))
        assert rep.iterations == ref["iterations"] and rep.converged == ref["converged"]
        assert rel_l2(rep.solution.values, ref["solution"]) <= 1e-7


# ---- full BASELINE sizes (digests of the reference's own runs) --------------------

@pytest.mark.slow
def test_cfg2_full_size():
    g = golden("cfg2_full")
    a = gen.cfg2_random_two_phase()
    reps = solve_batch(a, [LoadCase(E) for E in gen.CFG2_LOADS], SolverConfig(tol=1e-8, max_iter=2000))
    en = a.device().energy(np.array(gen.CFG2_LOADS), np.stack([r.solution.values for r in reps]))
    for j, rep in enumerate(reps):
        check_report(rep, g, f"l{j}_")
        assert abs(en[j, j] - float(g[f"l{j}_energy"])) <= AH_TOL * abs(float(g[f"l{j}_energy"]))


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg4_81", "cfg5_81"])
def test_down_scaled_cfg4_cfg5(name):
    g = golden(name)
    if name == "cfg4_81":
        a = gen.cfg4_polycrystal(81)
        load = (1.0, 0.0, 0.0)
    else:
        a = gen.cfg5_two_phase(81)
        load = gen.CFG5_LOAD
    rep = solve_cg(a, LoadCase(load), SolverConfig(tol=1e-8, max_iter=3000))
    check_report(rep, g, "cg_")
    en = a.device().energy(np.array([load]), rep.solution.values[None])
    assert abs(en[0, 0] - float(g["energy"])) <= AH_TOL * abs(float(g["energy"]))


@pytest.mark.slow
def test_cfg3_full_size():
    g = golden("cfg3_full")
    a = gen.cfg3_sphere()
    load = LoadCase((1.0, 0.0, 0.0))
    rep = solve_cg(a, load, SolverConfig(tol=1e-8, max_iter=2000))
    check_report(rep, g, "cg_")
    en = a.device().energy(np.array([load.E]), rep.solution.values[None])
    assert abs(en[0, 0] - float(g["cg_energy"])) <= AH_TOL * abs(float(g["cg_energy"]))
    if "fp_iterations" in g:
        check_report(solve_neumann(a, load, SolverConfig(method="neumann", tol=1e-6, max_iter=2000)), g, "fp_")


@pytest.mark.slow
def test_cfg5_405_full_size():
    """The single-GPU stand-in of BASELINE configs[4]: the cfg5 generator at 405^3
    (radix-5 register-FFT axis, contrast 1000) against a full solve of the
    unmodified reference (tests/golden/make_cfg5_405.py): iteration count,
    residual history, 4096 sampled solution values, energy."""
    g = golden("cfg5_405")
    a = gen.cfg5_two_phase(int(g["n"]))
    rep = solve_cg(a, LoadCase(gen.CFG5_LOAD), SolverConfig(tol=1e-8, max_iter=3000))
    check_report(rep, g, "cg_", case="cfg5_405")
    en = a.device().energy(np.array([gen.CFG5_LOAD]), rep.solution.values[None])
    assert abs(en[0, 0] - float(g["energy"])) <= AH_TOL * abs(float(g["energy"]))


def test_device_voronoi_generator_matches_host():
    """fc_generate_voronoi == generators.voronoi_labels bit for bit, and the poly27
    golden solve is reproduced from the device-generated field."""
    from paper_1311_0089_b200 import _native

    for n in (27, 45):
        seeds, packed = gen.cfg4_grains(512, gen.SEEDS["cfg4"], n)
        ctx = _native.Context(GridSpec((1.0,) * 3, (n,) * 3))
        labels = ctx.generate_voronoi(seeds, packed, want_labels=True)
        assert np.array_equal(labels, gen.voronoi_labels(n, seeds))
    g = golden("poly27")
    seeds, packed = gen.cfg4_grains(512, gen.SEEDS["cfg4"], 27)
    ctx = _native.Context(GridSpec((1.0,) * 3, (27,) * 3))
    ctx.generate_voronoi(seeds, packed)
    outs, x, _ = ctx.solve_cg(np.array([[1.0, 0.0, 0.0]]), 1e-8, 2000)
    assert outs[0]["iterations"] == int(g["cg_iterations"])
    assert rel_l2(x[0], g["cg_solution"]) <= max(SOL_TOL, 10 * float(g["cg_floor"]))


@pytest.mark.slow
def test_cfg4_full_size_anchor():
    """cfg4 at 729^3 (BASELINE configs[3]) against the first CG iterations of the
    CPU oracle at full size (tests/golden/make_cfg4_anchor.py):
    same generator (device labels), max_iter = 3, residual history r_0..r_3 within
    1e-12 relative, the 4096 sampled solution values within 1e-9 relative L2,
    energy within 1e-10 relative."""
    from paper_1311_0089_b200 import _native

    g = golden("cfg4_729_anchor")
    n = int(g["n"])
    seeds, packed = gen.cfg4_grains(512, gen.SEEDS["cfg4"], n)
    ctx = _native.Context(GridSpec((1.0,) * 3, (n,) * 3))
    ctx.generate_voronoi(seeds, packed)
    E = np.array([[1.0, 0.0, 0.0]])
    outs, x, _ = ctx.solve_cg(E, 1e-8, int(g["max_iter"]))
    assert outs[0]["iterations"] == int(g["iterations"])
    h = outs[0]["history"]
    ref_h = g["history"]
    hist_dev = float(np.max(np.abs(h - ref_h) / ref_h[0]))
    got = x[0].reshape(-1)[g["sample_idx"]]
    sample_err = rel_l2(got, g["sample"])
    en = ctx.energy(E)[0, 0]
    en_err = abs(en - float(g["energy"])) / abs(float(g["energy"]))
    log_parity({"case": "cfg4_729_anchor", "hist_dev": hist_dev, "sample_err": sample_err, "energy_err": en_err})
    assert hist_dev <= 1e-12, hist_dev
    assert sample_err <= SOL_TOL, sample_err
    assert en_err <= AH_TOL, en_err
