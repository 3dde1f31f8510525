"""Pin the CPU oracle (oracle/fftcell_oracle.py) against fixtures produced by
running the unmodified reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import golden, rel_l2
from oracle import fftcell_oracle as orc
from paper_1311_0089_b200 import generators as gen


def _full(packed, d):
    return orc.unpack(packed, d)


def test_operators_match_reference():
    g = golden("operators")
    for i in range(int(g["ncase"])):
        Y, shape = tuple(g[f"c{i}_Y"]), tuple(int(s) for s in g[f"c{i}_shape"])
        d = len(shape)
        full = _full(g[f"c{i}_packed"], d)
        u = g[f"c{i}_u"]
        proj = orc.Projector(shape, Y, g[f"c{i}_A0"])
        np.testing.assert_allclose(orc.apply_system(full, u, shape, Y), g[f"c{i}_system"], rtol=0, atol=1e-13)
        np.testing.assert_allclose(proj.apply_orthogonal(u), g[f"c{i}_orth"], rtol=0, atol=1e-13)
        np.testing.assert_allclose(proj.apply_gamma_ref(u), g[f"c{i}_gamma"], rtol=0, atol=1e-13)
        np.testing.assert_allclose(orc.apply_A(full, u), g[f"c{i}_Au"], rtol=0, atol=1e-13)


def test_cfg1_cg_fixed_point_and_effective_tensor():
    g = golden("cfg1")
    a = gen.cfg1_square_inclusion()
    full = orc.isotropic_full(a.components[0], 2)
    shape, Y = a.spec.shape, a.spec.half_periods
    cg = orc.solve_cg(full, (1.0, 0.0), shape, Y, 1e-8, 1000)
    assert cg["iterations"] == int(g["cg_iterations"]) == 21
    assert rel_l2(cg["solution"], g["cg_solution"]) < 1e-13
    np.testing.assert_allclose(cg["history"], g["cg_history"], rtol=1e-12)
    fp = orc.solve_neumann(full, (1.0, 0.0), shape, Y, 1e-8, 1000, float(g["fp_mean_lambda"]) * np.eye(2))
    assert fp["iterations"] == int(g["fpmean_iterations"]) == 18
    assert not fp["converged"] and fp["message"] == str(g["fpmean_message"])
    lo, hi = orc.bounds(full, 2)
    fpd = orc.solve_neumann(full, (1.0, 0.0), shape, Y, 1e-8, 1000, orc.default_reference_scalar(lo, hi) * np.eye(2))
    assert fpd["iterations"] == int(g["fpdef_iterations"]) == 59
    sols = [orc.solve_cg(full, e, shape, Y, 1e-8, 1000)["solution"] for e in np.eye(2)]
    np.testing.assert_allclose(orc.effective_tensor(full, shape, Y, sols), g["AH"], rtol=1e-13)


def test_sine_and_dense_cases():
    g = golden("sine255")
    full = _full(g["packed"], 1)
    sol = orc.solve_cg(full, (1.0,), (255,), (1.0,), 1e-10, 500)
    assert sol["iterations"] == int(g["cg_iterations"])
    AH = orc.effective_tensor(full, (255,), (1.0,), [sol["solution"]])
    assert abs(AH[0, 0] - float(g["AH"][0, 0])) < 1e-13
    assert abs(AH[0, 0] - np.sqrt(5.0)) <= 1e-6
    g = golden("dense_small")
    for i in range(int(g["ncase"])):
        shape, Y, E = tuple(int(s) for s in g[f"c{i}_shape"]), tuple(g[f"c{i}_Y"]), tuple(g[f"c{i}_E"])
        full = _full(g[f"c{i}_packed"], len(shape))
        rep = orc.solve_cg(full, E, shape, Y, 1e-13, 2000)
        assert rep["iterations"] == int(g[f"c{i}_iterations"])
        np.testing.assert_allclose(rep["solution"], g[f"c{i}_solution"], rtol=0, atol=1e-13)
        if len(shape) * np.prod(shape) <= 200:
            np.testing.assert_allclose(orc.dense_solve(full, E, shape, Y), g[f"c{i}_dense"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", ["sphere27", "poly27"])
def test_3d_cases(name):
    g = golden(name)
    if name == "sphere27":
        a = gen.cfg3_sphere(27)
        full = orc.isotropic_full(a.components[0], 3)
    else:
        full = _full(g["packed"], 3)
    shape, Y = (27, 27, 27), (1.0, 1.0, 1.0)
    cg = orc.solve_cg(full, (1.0, 0.0, 0.0), shape, Y, 1e-8, 2000)
    assert cg["iterations"] == int(g["cg_iterations"])
    assert rel_l2(cg["solution"], g["cg_solution"]) < 1e-12


def test_generators_match_survey_statistics():
    a = gen.cfg1_square_inclusion()
    assert abs(a.components[0].mean() - 4.29355281207133) < 1e-12
    assert abs((gen.cfg3_sphere(243).components[0] > 1).mean() - 0.1795581363793075) < 1e-15
    seeds, packed = gen.cfg4_grains(512, gen.SEEDS["cfg4"], 729)
    assert seeds.shape == (512, 3) and packed.shape == (512, 6)
    lam_min, lam_max = orc.eigen_range(orc.unpack(packed.T, 3), 3)
    assert np.all(lam_min > 0)


@pytest.mark.parametrize("name", ["poly27", "generic3d"])
def test_lean_cg_matches_reference_golden(name):
    """The memory-lean oracle (oracle/lean_cg.py: packed coefficients, half-spectrum
    FFT, BLAS dots) that produced the 729^3 anchor reproduces the reference's own
    solves: identical iteration counts, histories and solutions within the
    reference's rounding floor (poly27 is the ill-conditioned 27^3 polycrystal)."""
    from oracle import lean_cg

    g = golden(name)
    if name == "poly27":
        shape, Y, E, tol = (27, 27, 27), (1.0, 1.0, 1.0), (1.0, 0.0, 0.0), 1e-8
    else:
        shape, Y = tuple(int(s) for s in g["shape"]), tuple(g["Y"])
        E, tol = (0.3, -1.0, 0.5), 1e-9
    op = lean_cg.LeanOperator(shape, Y, packed=g["packed"])
    rep = lean_cg.solve_cg(op, E, tol, 2000)
    assert rep["iterations"] == int(g["cg_iterations"])
    h = np.array(rep["history"])
    ref = g["cg_history"]
    assert np.max(np.abs(h - ref) / ref[0]) <= max(1e-12, 10 * float(g["cg_floor_hist"]))
    assert np.max(np.abs(h[:4] - ref[:4]) / ref[0]) <= 1e-13  # the anchor's iterations
    assert rel_l2(rep["solution"], g["cg_solution"]) <= max(1e-9, 10 * float(g["cg_floor"]))


def test_cg_stepper_is_solve_cg():
    """bench.py's CPU sample (CGStepper) runs exactly solve_cg's iterations."""
    g = golden("poly27")
    st = orc.CGStepper(orc.unpack(g["packed"], 3), (1.0, 0.0, 0.0), (27,) * 3, (1.0,) * 3, 1e-8)
    st.setup()
    while st.step():
        pass
    assert st.iterations == int(g["cg_iterations"])
    np.testing.assert_array_equal(np.array(st.history), g["cg_history"])
