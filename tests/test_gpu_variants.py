"""GPU: every kernel variant of the row / outer sweeps gives the same CG solve.

The sweeps have alternative implementations selected by environment switches
read when a context is created (fc_engine.cu): TMA tensor boxes for the
transposed half spectrum (FC_ROW_TMA), bulk pencil copies in the outer sweep
(FC_OUTER_TMA), the persistent double-buffered last sweep (FC_INV_PIPE) and
first sweep (FC_ROW_PIPE).  They perform the same arithmetic in the same order,
so the batched solve must agree to the last bit with the default path; the
default path itself is checked against the CPU oracle.  A 243 x 2187 grid has
one-pencil row blocks (rows of 2187), the case the persistent kernels handle.
"""

import os

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


def _solve(a, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        ctx = _native.Context(GridSpec((1.0, 1.0), SHAPE))
        ctx.set_coefficients(_field(a))
        reps, x, _ = ctx.solve_cg(LOADS, 1e-8, 1000)
        return [r["iterations"] for r in reps], x
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


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


@pytest.mark.parametrize("env", [
    {"FC_ROW_TMA": "0"},
    {"FC_OUTER_TMA": "0"},
    {"FC_INV_PIPE": "0"},
    {"FC_ROW_PIPE": "1"},
    {"FC_ROW_PIPE": "1", "FC_INV_STAGES": "3"},
    {"FC_INV_QBUF": "0"},
    {"FC_OUTER_PERSIST": "1"},
    {"FC_OUTER_C1_2D": "1"},
    {"FC_DEFER_X": "0"},
    {"FC_DEFER_X": "0", "FC_ROW_PIPE": "1"},
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_variant_is_bitwise_identical(medium, default_solve, env):
    its0, x0 = default_solve
    its, x = _solve(medium, env)
    assert its == its0
    assert np.array_equal(x, x0), rel_l2(x, x0)


def test_mid_sweep_variants_3d():
    """3-D: the TMA middle sweep (FC_MID_TMA) and the outer CTA size
    (FC_OUTER_THREADS) give a bitwise-identical CG solve."""
    from paper_1311_0089_b200 import CoefficientField

    shape = (81, 81, 81)
    spec = GridSpec((1.0, 1.0, 1.0), shape)
    rng = np.random.default_rng(81)
    a = np.where(rng.random(shape) < 0.3, 50.0, 1.0)
    coef = CoefficientField.isotropic(spec, a)

    def run(env):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            ctx = _native.Context(spec)
            ctx.set_coefficients(coef)
            reps, x, _ = ctx.solve_cg(np.array([[1.0, 0.0, 0.0]]), 1e-8, 1000)
            return reps[0]["iterations"], x
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v

    it0, x0 = run({})
    for env in ({"FC_MID_TMA": "0"}, {"FC_OUTER_THREADS": "256"}, {"FC_OUTER_TMA": "0"}, {"FC_OUTER_SEQ": "1"}):
        it, x = run(env)
        assert it == it0, env
        assert np.array_equal(x, x0), (env, rel_l2(x, x0))


def test_anisotropic_first_sweep_variants():
    """Packed coefficients: the split first sweep (pointwise kernel + staged row
    FFT, default) and the all-components fused first sweep (FC_ANISO_SPLIT=0)
    give a bitwise-identical CG solve."""
    from conftest import random_spd_packed
    from paper_1311_0089_b200 import CoefficientField

    shape = (27, 27, 81)
    spec = GridSpec((1.0, 1.0, 1.0), shape)
    packed = random_spd_packed(shape, np.random.default_rng(27))
    coef = CoefficientField(spec, packed)

    def run(env):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            ctx = _native.Context(spec)
            ctx.set_coefficients(coef)
            reps, x, _ = ctx.solve_cg(np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 1.0]]), 1e-8, 1000)
            return [r["iterations"] for r in reps], x
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v

    it0, x0 = run({})
    it1, x1 = run({"FC_ANISO_SPLIT": "0"})
    assert it0 == it1
    assert np.array_equal(x0, x1), rel_l2(x1, x0)


def _env_run(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("case", ["iso2d_3k", "iso2d_generic", "aniso3d", "aniso3d_fused", "line1d"])
@pytest.mark.parametrize("max_iter", [4, 1000])
def test_deferred_x_update_is_bitwise_identical(case, max_iter):
    """The CG x update deferred into the next first sweep (FC_DEFER_X=1, the
    default) and flushed after the loop gives the same solution bits as the
    immediate update in k_cg_update, for RHSs stopping at different iterations,
    at max_iter, and on every first-sweep kernel (register / generic / split and
    fused anisotropic / 1-D line)."""
    from conftest import random_spd_packed
    from paper_1311_0089_b200 import CoefficientField

    rng = np.random.default_rng(7)
    env = {}
    if case == "iso2d_3k":
        shape, loads = (81, 243), np.array([[1.0, 0.0], [0.0, 1.0], [0.6, 0.8]])
        coef_fn = lambda spec: CoefficientField.isotropic(spec, np.where(rng.random(shape) < 0.4, 30.0, 1.0))
    elif case == "iso2d_generic":
        shape, loads = (25, 35), np.array([[1.0, 0.0], [0.0, 1.0]])
        coef_fn = lambda spec: CoefficientField.isotropic(spec, np.where(rng.random(shape) < 0.4, 30.0, 1.0))
    elif case in ("aniso3d", "aniso3d_fused"):
        shape, loads = (27, 27, 81), np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
        coef_fn = lambda spec: CoefficientField(spec, random_spd_packed(shape, rng))
        if case == "aniso3d_fused":
            env = {"FC_ANISO_SPLIT": "0"}
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

    r1, x1 = _env_run({**env, "FC_DEFER_X": "1"}, run)
    r0, x0 = _env_run({**env, "FC_DEFER_X": "0"}, run)
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

    i1, x1 = _env_run({}, run)
    i0, x0 = _env_run({"FC_OUTER_SEQ": "0"}, run)
    assert i1 == i0 == 52
    assert np.array_equal(x1, x0), rel_l2(x1, x0)
