"""GPU: every kernel variant of the sweeps gives the same CG solve.

The sweeps have alternative implementations selected by plan options frozen
into a context at creation (fc_set_plan_option, include/fftcell_b200.h): TMA
tensor boxes for the transposed half spectrum (row_tma), bulk pencil copies in
the outer sweep (outer_tma), the persistent double-buffered last sweep
(inv_pipe), the fused packed first sweep (aniso_fused), the deferred x update
(defer_x).  They perform the same arithmetic in the same order, so the batched
solve must agree to the last bit with the default path; the default path
itself is checked against the CPU oracle.  A 243 x 2187 grid has one-pencil row
blocks (rows of 2187), the case the persistent kernels handle.
"""

import numpy as np
import pytest

from conftest import rel_l2
from oracle import fftcell_oracle as orc
from paper_1311_0089_b200 import _native
from paper_1311_0089_b200.grid import GridSpec

pytestmark = pytest.mark.gpu

SHAPE = (243, 2187)
LOADS = np.array([[1.0, 0.0], [0.6, 0.8]])


def _medium():
    rng = np.random.default_rng(243)
    noise = rng.standard_normal(SHAPE)
    f0 = np.fft.fftfreq(SHAPE[0])[:, None]
    f1 = np.fft.fftfreq(SHAPE[1])[None, :]
    smooth = np.fft.ifft2(np.fft.fft2(noise) * np.exp(-2 * np.pi**2 * 9.0 * (f0**2 + f1**2))).real
    return np.where(smooth > np.quantile(smooth, 0.6), 100.0, 1.0)


def _solve(a, opts):
    with _native.plan_options(**opts):
        ctx = _native.Context(GridSpec((1.0, 1.0), SHAPE))
    ctx.set_coefficients(_field(a))
    reps, x, _ = ctx.solve_cg(LOADS, 1e-8, 1000)
    return [r["iterations"] for r in reps], x


def _field(a):
    from paper_1311_0089_b200 import CoefficientField

    return CoefficientField.isotropic(GridSpec((1.0, 1.0), SHAPE), a)


@pytest.fixture(scope="module")
def medium():
    return _medium()


@pytest.fixture(scope="module")
def default_solve(medium):
    return _solve(medium, {})


def test_default_path_matches_oracle(medium, default_solve):
    its, x = default_solve
    full = orc.isotropic_full(medium, 2)
    ref = orc.solve_cg(full, tuple(LOADS[0]), SHAPE, (1.0, 1.0), 1e-8, 1000)
    assert its[0] == ref["iterations"]
    assert rel_l2(x[0], ref["solution"]) < 1e-9


@pytest.mark.parametrize("opts", [
    {"row_tma": 0},
    {"outer_tma": 0},
    {"inv_pipe": 0},
    {"defer_x": 0},
    {"defer_x": 0, "inv_pipe": 0},
    {"outer_seq": 1},
    {"outer_seq": 0},
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_variant_is_bitwise_identical(medium, default_solve, opts):
    its0, x0 = default_solve
    its, x = _solve(medium, opts)
    assert its == its0
    assert np.array_equal(x, x0), rel_l2(x, x0)


@pytest.mark.parametrize("shape", [(81, 81, 81), (27, 729, 45)])
def test_mid_sweep_variants_3d(shape):
    """3-D: the TMA middle sweeps (mid_tma, mid_tma_fwd), their thread mapping
    (mid_map) and CTA sizes (mid_threads, mid_threads_inv), the outer CTA size
    (outer_threads), the outer bulk copies and the one-component outer sweep
    give a bitwise-identical CG solve."""
    from paper_1311_0089_b200 import CoefficientField

    spec = GridSpec((1.0, 1.0, 1.0), shape)
    rng = np.random.default_rng(81)
    a = np.where(rng.random(shape) < 0.3, 50.0, 1.0)
    coef = CoefficientField.isotropic(spec, a)

    def run(opts):
        with _native.plan_options(**opts):
            ctx = _native.Context(spec)
        ctx.set_coefficients(coef)
        reps, x, _ = ctx.solve_cg(np.array([[1.0, 0.0, 0.0]]), 1e-8, 1000)
        return reps[0]["iterations"], x

    it0, x0 = run({})
    for opts in ({"two_field": 0}, {"fold_fwd": 0}, {"fold_fwd": 1}, {"mid_tma": 0}, {"outer_threads": 256}, {"outer_tma": 0}, {"outer_seq": 1}, {"outer_seq": 0}, {"mid_map": 0},
                 {"mid_tma_fwd": 0}, {"mid_map": 0, "mid_tma_fwd": 0}, {"mid_threads": 512, "mid_threads_inv": 512},
                 {"mid_threads": 81, "mid_threads_inv": 162}):
        it, x = run(opts)
        assert it == it0, opts
        assert np.array_equal(x, x0), (opts, rel_l2(x, x0))


@pytest.mark.parametrize("shape", [(81, 81, 27), (243, 81, 81), (45, 135, 27), (729, 243, 9), (35, 243, 81)])
def test_two_field_sweeps_match_three_field(shape):
    """d = 3, one slab: the outer sweep stores t = F0^-1 q once instead of xi1 t and
    xi2 t, and the inverse middle sweep rebuilds both components from it as it loads
    them (two_field = 1, the default: 8 bytes per voxel less written and, with the two
    components' CTAs side by side, read).  Same products in the same order as the
    three-field sweeps: CG with several loads, the fixed point and both projectors
    agree bit for bit.  Shapes: power-of-three and radix-5 middle and outer axes,
    ragged pencil blocks, and an outer axis off the register path (35: two_field
    stays off, the option must be harmless)."""
    from conftest import random_spd_packed
    from paper_1311_0089_b200 import CoefficientField

    spec = GridSpec((1.0, 0.7, 1.3), shape)
    rng = np.random.default_rng(5)
    coef = CoefficientField(spec, random_spd_packed(shape, rng))
    E = np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.3, 0.4, 0.5]])
    u = rng.standard_normal((2, 3) + shape)
    ref = np.array([[2.0, 0.3, 0.1], [0.3, 3.0, 0.2], [0.1, 0.2, 4.0]])

    def run(opts):
        with _native.plan_options(**opts):
            ctx = _native.Context(spec)
        ctx.set_coefficients(coef)
        reps, x, hist = ctx.solve_cg(E, 1e-8, 60)
        freps, fx = ctx.solve_fixed_point(E[:2], 1e-6, 25, np.diag([4.0, 5.0, 6.0]), np.ones(2))
        return ([r["iterations"] for r in reps], x, hist, [r["iterations"] for r in freps], fx,
                ctx.project(0, None, u), ctx.project(1, ref, u), ctx.apply_system(u))

    three = run({"two_field": 0})
    for opts in ({}, {"fold_fwd": 0}, {"fold_fwd": 1}):
        two = run(opts)
        assert two[0] == three[0] and two[3] == three[3], opts
        for k in (1, 2, 4, 5, 6, 7):
            assert np.array_equal(two[k], three[k]), (opts, k, rel_l2(two[k], three[k]))


@pytest.mark.parametrize("shape", [(27, 27, 81), (81, 81, 729), (45, 27, 405)])
def test_anisotropic_first_sweep_variants(shape):
    """Packed coefficients: the fused first sweep (pointwise step and row FFT of
    all components in one CTA, default) and the split variant (pointwise kernel
    writing y, then the staged row FFT; aniso_fused = 0) give a bitwise-identical
    CG solve and fixed point; rows of 81, 729 (cfg4) and 405 (radix-5)."""
    from conftest import random_spd_packed
    from paper_1311_0089_b200 import CoefficientField

    spec = GridSpec((1.0, 1.0, 1.0), shape)
    packed = random_spd_packed(shape, np.random.default_rng(27))
    coef = CoefficientField(spec, packed)
    E = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])

    def run(opts):
        with _native.plan_options(**opts):
            ctx = _native.Context(spec)
        ctx.set_coefficients(coef)
        reps, x, _ = ctx.solve_cg(E, 1e-8, 1000)
        A0 = np.diag([4.0, 5.0, 6.0])
        freps, fx = ctx.solve_fixed_point(E, 1e-6, 40, A0, np.ones(2))
        return [r["iterations"] for r in reps], x, [r["iterations"] for r in freps], fx

    it0, x0, fi0, fx0 = run({})
    it1, x1, fi1, fx1 = run({"aniso_fused": 0})
    assert it0 == it1
    assert np.array_equal(x0, x1), rel_l2(x1, x0)
    assert fi0 == fi1
    assert np.array_equal(fx0, fx1), rel_l2(fx1, fx0)


def _opt_run(opts, fn):
    with _native.plan_options(**opts):
        return fn()


@pytest.mark.parametrize("case", ["iso2d_3k", "iso2d_generic", "aniso3d", "aniso3d_split", "line1d"])
@pytest.mark.parametrize("max_iter", [4, 1000])
def test_deferred_x_update_is_bitwise_identical(case, max_iter):
    """The CG x update deferred into the next first sweep (defer_x = 1, the
    default) and flushed after the loop gives the same solution bits as the
    immediate update in k_cg_update, for RHSs stopping at different iterations,
    at max_iter, and on every first-sweep kernel (register / generic / fused and
    split anisotropic / 1-D line)."""
    from conftest import random_spd_packed
    from paper_1311_0089_b200 import CoefficientField

    rng = np.random.default_rng(7)
    opts = {}
    if case == "iso2d_3k":
        shape, loads = (81, 243), np.array([[1.0, 0.0], [0.0, 1.0], [0.6, 0.8]])
        coef_fn = lambda spec: CoefficientField.isotropic(spec, np.where(rng.random(shape) < 0.4, 30.0, 1.0))
    elif case == "iso2d_generic":
        shape, loads = (25, 35), np.array([[1.0, 0.0], [0.0, 1.0]])
        coef_fn = lambda spec: CoefficientField.isotropic(spec, np.where(rng.random(shape) < 0.4, 30.0, 1.0))
    elif case in ("aniso3d", "aniso3d_split"):
        shape, loads = (27, 27, 81), np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
        coef_fn = lambda spec: CoefficientField(spec, random_spd_packed(shape, rng))
        if case == "aniso3d_split":
            opts = {"aniso_fused": 0}
    else:
        # continuous values: with two phases 1-D CG stops after 2 iterations
        shape, loads = (243,), np.array([[1.0]])
        coef_fn = lambda spec: CoefficientField.isotropic(spec, 1.0 + 30.0 * rng.random(shape))
    spec = GridSpec((1.0,) * len(shape), shape)
    coef = coef_fn(spec)

    def run():
        ctx = _native.Context(spec)
        ctx.set_coefficients(coef)
        reps, x, _ = ctx.solve_cg(loads, 1e-8, max_iter)
        return [(r["iterations"], r["converged"]) for r in reps], x

    r1, x1 = _opt_run({**opts, "defer_x": 1}, run)
    r0, x0 = _opt_run({**opts, "defer_x": 0}, run)
    assert r1 == r0
    assert np.array_equal(x1, x0), rel_l2(x1, x0)
    if max_iter == 4:
        assert all(it == 4 and not conv for it, conv in r1)


def test_outer_sequential_default_at_243():
    """243^3 (cfg3 size) runs the one-component-at-a-time outer sweep by
    default; it must give the same bits as the register version."""
    from paper_1311_0089_b200 import generators as gen

    a = gen.cfg3_sphere(243)
    E = np.array([[1.0, 0.0, 0.0]])

    def run():
        ctx = _native.Context(a.spec)
        ctx.set_coefficients(a)
        reps, x, _ = ctx.solve_cg(E, 1e-8, 1000)
        return reps[0]["iterations"], x

    i1, x1 = _opt_run({}, run)
    i0, x0 = _opt_run({"outer_seq": 0}, run)
    assert i1 == i0 == 52
    assert np.array_equal(x1, x0), rel_l2(x1, x0)
