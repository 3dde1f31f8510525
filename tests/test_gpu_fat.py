"""GPU: the fat-thread outer sweep (plan option outer_fat: 27 values per thread,
warp-owned pencils, fc_kernels_fat.cuh), the split finalize (fin_split) and the
staged epilogue input of the last sweep (inv_qpre).

The fat-thread transform factors the axis differently (radix 27 instead of 9), so
it agrees with the default path to rounding, not bitwise: operators against the
CPU oracle at 1e-12, CG solves with equal iteration counts.  The split finalize
sums the same partials in another fixed order (same criterion).  inv_qpre moves
the same values through shared memory: bitwise.
"""

import numpy as np
import pytest

from conftest import rel_l2
from oracle import fftcell_oracle as orc
from paper_1311_0089_b200 import CoefficientField, _native
from paper_1311_0089_b200.grid import GridSpec

pytestmark = pytest.mark.gpu


def _ctx(shape, a, opts=None, cell=None):
    spec = GridSpec(cell or (1.0,) * len(shape), shape)
    with _native.plan_options(**(opts or {})):
        ctx = _native.Context(spec)
    ctx.set_coefficients(CoefficientField.isotropic(spec, a))
    return ctx


def _medium(shape, seed):
    rng = np.random.default_rng(seed)
    return np.where(rng.random(shape) < 0.35, 25.0, 1.0)


# outer axis (axis 0) on every fat length; the other axes on any path
FAT_SHAPES = [(27, 45), (81, 81), (243, 27), (729, 45), (2187, 27), (27, 9, 15), (81, 27, 9), (243, 9, 27), (729, 9, 9)]


@pytest.mark.parametrize("shape", FAT_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_fat_outer_operator_matches_oracle(shape):
    a = _medium(shape, 1)
    d = len(shape)
    cell = tuple(1.0 + 0.25 * i for i in range(d))
    u = np.random.default_rng(2).standard_normal((2, d) + shape)
    got = _ctx(shape, a, {"outer_fat": 1}, cell).apply_system(u)
    base = _ctx(shape, a, None, cell).apply_system(u)
    for k in range(2):
        ref = orc.apply_system(orc.isotropic_full(a, d), u[k], shape, cell)
        assert np.max(np.abs(got[k] - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert rel_l2(got, base) <= 1e-13


def test_fat_outer_constant_field_projects_to_zero():
    # difference-form butterflies: constants give exact zeros in every non-DC mode
    shape = (729, 27)
    ctx = _ctx(shape, np.ones(shape), {"outer_fat": 1})
    u = np.empty((1, 2) + shape)
    u[0, 0] = 3.0
    u[0, 1] = -1.5
    assert not np.any(ctx.apply_system(u))


@pytest.mark.parametrize("shape", [(243, 81), (81, 27, 27)], ids=lambda s: "x".join(map(str, s)))
def test_fat_outer_cg_matches_oracle(shape):
    a = _medium(shape, 3)
    d = len(shape)
    E = np.eye(d)[:1]
    reps, x, _ = _ctx(shape, a, {"outer_fat": 1}).solve_cg(E, 1e-8, 1000)
    ref = orc.solve_cg(orc.isotropic_full(a, d), tuple(E[0]), shape, (1.0,) * d, 1e-8, 1000)
    assert reps[0]["iterations"] == ref["iterations"]
    assert rel_l2(x[0], ref["solution"]) < 1e-9


@pytest.mark.parametrize("shape", [(243, 243), (81, 81, 27)], ids=lambda s: "x".join(map(str, s)))
def test_split_finalize_matches_fused(shape):
    a = _medium(shape, 5)
    d = len(shape)
    E = np.eye(d)[:2]
    r0, x0, _ = _ctx(shape, a, {"fin_split": 0}).solve_cg(E, 1e-8, 1000)
    r1, x1, _ = _ctx(shape, a, {"fin_split": 1}).solve_cg(E, 1e-8, 1000)
    assert [r["iterations"] for r in r0] == [r["iterations"] for r in r1]
    assert rel_l2(x1, x0) < 1e-12
    for q0, q1 in zip(r0, r1):
        assert np.allclose(q0["history"], q1["history"], rtol=1e-10, atol=0.0)
    A0 = np.diag(np.full(d, 13.0))
    scale = [1.0, 1.0]
    f0 = _ctx(shape, a, {"fin_split": 0}).solve_fixed_point(E, 1e-6, 500, A0, scale)
    f1 = _ctx(shape, a, {"fin_split": 1}).solve_fixed_point(E, 1e-6, 500, A0, scale)
    assert [r["iterations"] for r in f0[0]] == [r["iterations"] for r in f1[0]]
    assert rel_l2(f1[1], f0[1]) < 1e-12


@pytest.mark.parametrize("shape", [(81, 243), (27, 81, 243), (9, 27, 729)], ids=lambda s: "x".join(map(str, s)))
def test_staged_epilogue_input_is_bitwise_identical(shape):
    a = _medium(shape, 7)
    d = len(shape)
    E = np.eye(d)[:2]
    r0, x0, _ = _ctx(shape, a, {"inv_qpre": 0}).solve_cg(E, 1e-8, 1000)
    r1, x1, _ = _ctx(shape, a, {"inv_qpre": 1}).solve_cg(E, 1e-8, 1000)
    assert [r["iterations"] for r in r0] == [r["iterations"] for r in r1]
    assert np.array_equal(x0, x1)
    A0 = np.diag(np.full(d, 13.0))
    f0 = _ctx(shape, a, {"inv_qpre": 0}).solve_fixed_point(E, 1e-6, 500, A0, [1.0, 1.0])
    f1 = _ctx(shape, a, {"inv_qpre": 1}).solve_fixed_point(E, 1e-6, 500, A0, [1.0, 1.0])
    assert [r["iterations"] for r in f0[0]] == [r["iterations"] for r in f1[0]]
    assert np.array_equal(f0[1], f1[1])


@pytest.mark.parametrize("shape", [(81, 27, 27), (243, 9, 27), (729, 9, 9), (405, 9, 15)], ids=lambda s: "x".join(map(str, s)))
def test_unstaged_outer_sweep_is_bitwise_identical(shape):
    # k_outer_dir: same transforms and g3_* arithmetic as the staged kernels, loads / stores straight from registers
    a = _medium(shape, 11)
    u = np.random.default_rng(12).standard_normal((2, 3) + shape)
    base = _ctx(shape, a).apply_system(u)
    got = _ctx(shape, a, {"outer_direct": 1}).apply_system(u)
    assert np.array_equal(got, base)
    E = np.eye(3)[:2]
    r0, x0, _ = _ctx(shape, a).solve_cg(E, 1e-8, 1000)
    r1, x1, _ = _ctx(shape, a, {"outer_direct": 1}).solve_cg(E, 1e-8, 1000)
    assert [r["iterations"] for r in r0] == [r["iterations"] for r in r1]
    assert np.array_equal(x0, x1)
