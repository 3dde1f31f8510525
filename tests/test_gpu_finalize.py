"""GPU: the split finalize (plan option fin_split) and the staged epilogue input
of the last sweep (inv_qpre).

The split finalize sums the same per-CTA partials in another fixed order, so it
agrees with the fused last-CTA finalize to rounding: equal iteration counts,
solutions within 1e-12, histories within 1e-6 (CG amplifies the difference
along the iterations).  inv_qpre moves the same values
through shared memory: bitwise.
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
        # CG amplifies the rounding difference of the two summation orders along the iterations
        assert np.allclose(q0["history"], q1["history"], rtol=1e-6, atol=0.0)
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

