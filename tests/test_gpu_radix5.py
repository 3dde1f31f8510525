"""GPU: register-path FFT lengths 5 * 3^k (45, 135, 405, 1215 -- the cfg5 axis
class).  Operators and CG solves against the CPU oracle, against the Stockham
path (plan option force_generic), and sharded against a single slab."""


import numpy as np
import pytest

from conftest import rel_l2
from oracle import fftcell_oracle as orc
from paper_1311_0089_b200 import CoefficientField, _native
from paper_1311_0089_b200.grid import GridSpec

pytestmark = pytest.mark.gpu


def _ctx(shape, a, opts=None, slabs=None):
    spec = GridSpec((1.0,) * len(shape), shape)
    with _native.plan_options(**(opts or {})):
        ctx = _native.Context(spec, slabs=slabs) if slabs else _native.Context(spec)
    ctx.set_coefficients(CoefficientField.isotropic(spec, a))
    return ctx


def _medium(shape, seed):
    rng = np.random.default_rng(seed)
    return np.where(rng.random(shape) < 0.35, 25.0, 1.0)


@pytest.mark.parametrize("shape", [(45, 1215), (1215, 45), (405, 135), (45, 135, 45), (135, 45, 405)])
def test_operator_matches_oracle(shape):
    a = _medium(shape, 1)
    d = len(shape)
    u = np.random.default_rng(2).standard_normal((d,) + shape)
    got = _ctx(shape, a).apply_system(u)
    ref = orc.apply_system(orc.isotropic_full(a, d), u, shape, (1.0,) * d)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("shape", [(45, 1215), (405, 135), (45, 135, 45)])
def test_cg_matches_oracle_and_generic(shape):
    a = _medium(shape, 3)
    d = len(shape)
    E = np.eye(d)[:1]
    reps, x, _ = _ctx(shape, a).solve_cg(E, 1e-8, 1000)
    ref = orc.solve_cg(orc.isotropic_full(a, d), tuple(E[0]), shape, (1.0,) * d, 1e-8, 1000)
    assert reps[0]["iterations"] == ref["iterations"]
    assert rel_l2(x[0], ref["solution"]) < 1e-9
    rg, xg, _ = _ctx(shape, a, {"force_generic": 1}).solve_cg(E, 1e-8, 1000)
    assert rg[0]["iterations"] == reps[0]["iterations"]
    assert rel_l2(xg, x) < 1e-12


@pytest.mark.parametrize("P", [2, 3])
def test_sharded_radix5(P):
    shape = (45, 45, 135)
    a = _medium(shape, 4)
    E = np.array([[0.0, 0.0, 1.0]])
    r1, x1, _ = _ctx(shape, a).solve_cg(E, 1e-8, 1000)
    rP, xP, _ = _ctx(shape, a, slabs=[0] * P).solve_cg(E, 1e-8, 1000)
    assert r1[0]["iterations"] == rP[0]["iterations"]
    assert rel_l2(xP, x1) <= 1e-12
