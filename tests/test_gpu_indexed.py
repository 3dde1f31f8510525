"""GPU: phase-indexed coefficients give the packed field's results bit for bit.

A piecewise-constant packed field (every BASELINE microstructure is one) can
live in HBM as one 16-bit label per voxel plus a table of its distinct packed
tensors (fc_set_coefficients_indexed from the host, fc_compress_coefficients
from a packed field already on the device).  The fused packed first sweep and
coef() then read the tensor through the label; the values are those of the
packed field (material.py:90-158), so solves, energies and pointwise products
must agree to the last bit with the packed upload, which itself is checked
against the CPU oracle.
"""

import numpy as np
import pytest

from conftest import rel_l2
from oracle import fftcell_oracle as orc
from paper_1311_0089_b200 import CoefficientField, MaterialDataError, _native
from paper_1311_0089_b200.grid import GridSpec

pytestmark = pytest.mark.gpu


def _spd(rng, n, d):
    q = rng.standard_normal((n, d, d))
    return q @ np.swapaxes(q, 1, 2) + 0.3 * np.eye(d)


def _blocks(rng, shape, nph, cell):
    """Labels constant on cell-sized bricks (ragged at the upper faces)."""
    coarse = rng.integers(0, nph, size=tuple(-(-n // cell) for n in shape))
    lab = coarse
    for ax, n in enumerate(shape):
        lab = np.repeat(lab, cell, axis=ax).take(range(n), axis=ax)
    return lab


def _case(shape, nph, cell, seed):
    rng = np.random.default_rng(seed)
    d = len(shape)
    spec = GridSpec((1.0,) * d, shape)
    tensors = _spd(rng, nph, d)
    labels = _blocks(rng, shape, nph, cell)
    labels.flat[:nph] = np.arange(nph)  # every phase present
    return spec, labels, tensors


def _ctx(spec, **opts):
    with _native.plan_options(**opts):
        return _native.Context(spec)


def _cg(ctx, E):
    reps, x, hist = ctx.solve_cg(E, 1e-8, 500)
    return [r["iterations"] for r in reps], x, hist


CASES = {
    "81^3/40": ((81, 81, 81), 40, 9, 1),
    "27x81x243/7": ((27, 81, 243), 7, 5, 2),
    "243^2/300": ((243, 243), 300, 4, 3),
    "45x81x27/5": ((45, 81, 27), 5, 6, 4),  # radix-5 axis 0 and a register row axis
}


@pytest.mark.parametrize("name", list(CASES))
def test_indexed_and_compressed_match_packed_bitwise(name):
    spec, labels, tensors = _case(*CASES[name])
    d = spec.dim
    a = CoefficientField.from_phases(spec, labels, tensors)
    assert a.phases is not None
    E = np.eye(d)[:2]
    ref = _ctx(spec)
    ref.set_coefficients(a, compress=False)
    assert ref.n_phases == 0
    its0, x0, h0 = _cg(ref, E)
    A0 = ref.energy(E)

    idx = _ctx(spec)
    idx.set_coefficients(a)  # labels + table from the host
    assert idx.n_phases == tensors.shape[0]
    its1, x1, h1 = _cg(idx, E)
    assert its1 == its0
    assert np.array_equal(x1, x0), rel_l2(x1, x0)
    assert np.array_equal(h1, h0)
    assert np.array_equal(idx.energy(E), A0)

    plain = CoefficientField(spec, a.components)  # no phase information: device deduplication
    cmp_ = _ctx(spec)
    cmp_.set_coefficients(plain)
    assert cmp_.n_phases == len(np.unique(a.components.reshape(a.components.shape[0], -1), axis=1).T)
    its2, x2, h2 = _cg(cmp_, E)
    assert its2 == its0
    assert np.array_equal(x2, x0), rel_l2(x2, x0)
    assert np.array_equal(cmp_.energy(E), A0)


def test_indexed_matches_oracle():
    spec, labels, tensors = _case((27, 27, 27), 6, 4, 11)
    a = CoefficientField.from_phases(spec, labels, tensors)
    ctx = _ctx(spec)
    ctx.set_coefficients(a)
    assert ctx.n_phases == 6
    its, x, _ = _cg(ctx, np.array([[1.0, 0.0, 0.0]]))
    ref = orc.solve_cg(orc.unpack(a.components, 3), (1.0, 0.0, 0.0), spec.shape, (1.0, 1.0, 1.0), 1e-8, 500)
    assert its[0] == ref["iterations"]
    assert rel_l2(x[0], ref["solution"]) < 1e-9


def test_indexed_consumers_of_the_full_field():
    """apply_A and the energy read through the labels; the bounds and the split /
    generic first sweeps rebuild the packed field on demand."""
    spec, labels, tensors = _case((27, 45, 27), 9, 3, 5)
    a = CoefficientField.from_phases(spec, labels, tensors)
    rng = np.random.default_rng(0)
    u = rng.standard_normal((3,) + spec.shape)
    ref = _ctx(spec)
    ref.set_coefficients(a, compress=False)
    idx = _ctx(spec)
    idx.set_coefficients(a)
    assert np.array_equal(idx.apply_A(u), ref.apply_A(u))
    lo, hi, at = idx.coefficient_bounds()
    assert (lo, hi, at) == ref.coefficient_bounds()
    assert lo == pytest.approx(a.c_A, rel=1e-13) and hi == pytest.approx(a.C_A, rel=1e-13)
    E = np.array([[0.0, 1.0, 0.0]])
    its0, x0, _ = _cg(ref, E)
    for opts in ({"aniso_fused": 0}, {"force_generic": 1}):
        alt = _ctx(spec, **opts)
        alt.set_coefficients(a)
        assert alt.n_phases == 9
        its, x, _ = _cg(alt, E)
        assert its == its0
        ref_alt = _ctx(spec, **opts)
        ref_alt.set_coefficients(a, compress=False)
        assert np.array_equal(x, _cg(ref_alt, E)[1])


def test_indexed_fixed_point_matches_packed():
    spec, labels, tensors = _case((81, 27, 27), 4, 7, 8)
    a = CoefficientField.from_phases(spec, labels, tensors)
    A0 = 0.5 * (a.c_A + a.C_A) * np.eye(3)
    E = np.array([[1.0, 0.0, 0.0]])
    out = []
    for compress in (False, True):
        ctx = _ctx(spec)
        ctx.set_coefficients(a, compress=compress)
        reps, x = ctx.solve_fixed_point(E, 1e-6, 2000, A0, 1.0)
        out.append((reps[0]["iterations"], x))
    assert out[0][0] == out[1][0] > 1
    assert np.array_equal(out[0][1], out[1][1])


def test_per_voxel_field_stays_packed():
    spec = GridSpec((1.0, 1.0, 1.0), (27, 27, 27))
    rng = np.random.default_rng(3)
    mats = np.moveaxis(_spd(rng, 27**3, 3).reshape(27, 27, 27, 3, 3), (3, 4), (0, 1))
    a = CoefficientField.from_matrices(spec, mats)
    ctx = _ctx(spec)
    ctx.set_coefficients(a)  # 19683 distinct tensors > FC_MAX_PHASES
    assert ctx.n_phases == 0
    its, x, _ = _cg(ctx, np.array([[1.0, 0.0, 0.0]]))
    ref = _ctx(spec)
    ref.set_coefficients(a, compress=False)
    assert np.array_equal(x, _cg(ref, np.array([[1.0, 0.0, 0.0]]))[1])
    assert ctx.compress_coefficients(max_phases=8) == 0


def test_indexed_on_slabs_matches_single():
    spec, labels, tensors = _case((81, 27, 81), 30, 6, 9)
    a = CoefficientField.from_phases(spec, labels, tensors)
    E = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    one = _ctx(spec)
    one.set_coefficients(a, compress=False)
    its0, x0, _ = _cg(one, E)
    for how in ("indexed", "compressed"):
        many = _native.Context(spec, slabs=[0, 0, 0])
        many.set_coefficients(a if how == "indexed" else CoefficientField(spec, a.components))
        assert many.n_phases >= 1
        its, x, _ = _cg(many, E)
        assert its == its0
        # slabs reduce their inner products slab by slab: same iterates to rounding
        assert rel_l2(x, x0) < 1e-12
        assert np.allclose(many.energy(E), one.energy(E), rtol=1e-13, atol=0)


def test_indexed_errors():
    spec, labels, tensors = _case((27, 27, 27), 5, 4, 2)
    table = CoefficientField.from_phases(spec, labels, tensors).phases[1]
    ctx = _ctx(spec)
    bad = labels.astype(np.uint16).copy()
    bad[3, 4, 5] = 5
    with pytest.raises(ValueError, match="label out of range"):
        ctx.set_coefficients_indexed(bad, table)
    with pytest.raises(ValueError, match="coefficients not set"):
        ctx.solve_cg(np.array([[1.0, 0.0, 0.0]]), 1e-8, 10)
    with pytest.raises(ValueError, match="label count"):
        ctx.set_coefficients_indexed(bad[:-1], table)
    with pytest.raises(ValueError):
        ctx.set_coefficients_indexed(bad, table[:-1])
    with pytest.raises(MaterialDataError):
        CoefficientField.from_phases(spec, labels + 1, tensors)
