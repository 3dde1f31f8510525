"""Host-side logic of the package (CPU only): validation and error behaviour
mirroring the reference (grid.py, material.py, solver.py, green.py), voxel IO,
and the C ABI surface of the CUDA library."""

import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT, random_spd_packed
from paper_1311_0089_b200 import (
    CoefficientField, GridField, GridSpec, LoadCase, MaterialDataError, ReferenceTensor, SolverConfig,
    VoxelFormatError, load_field, load_voxel, save_coefficients, save_field,
)
from paper_1311_0089_b200 import _native, material


def test_even_grid_rejected():
    with pytest.raises(ValueError, match="odd"):
        GridSpec((1.0, 1.0), (4, 5))


def test_config_validation_and_alias():
    for kw in ({"method": "sor"}, {"tol": 1.0}, {"tol": 0.0}, {"max_iter": 0}):
        with pytest.raises(ValueError):
            SolverConfig(**kw)
    assert SolverConfig(method="fixed_point").method == "neumann"
    with pytest.raises(ValueError, match="scalar"):
        SolverConfig(method="cg", reference=ReferenceTensor(np.diag([2.0, 1.0])))


def test_load_case_validation():
    with pytest.raises(ValueError, match="finite"):
        LoadCase((1.0, np.inf))
    with pytest.raises(ValueError, match="dimension"):
        LoadCase((1.0,)).expand(GridSpec((1.0, 1.0), (3, 3)))


def test_material_bounds_match_oracle(rng):
    from oracle import fftcell_oracle as orc

    for shape in [(9,), (5, 7), (3, 5, 7)]:
        spec = GridSpec((1.0,) * len(shape), shape)
        packed = random_spd_packed(shape, rng)
        a = CoefficientField(spec, packed)
        lo, hi = orc.bounds(orc.unpack(packed, len(shape)), len(shape))
        assert a.c_A == lo and a.C_A == hi
        assert a.isotropic_values is None or len(shape) == 1


def test_isotropic_detection_and_bounds():
    spec = GridSpec((1.0, 1.0, 1.0), (3, 5, 7))
    vals = np.where(np.arange(105).reshape(3, 5, 7) % 2 == 0, 1.0, 50.0)
    a = CoefficientField.isotropic(spec, vals)
    assert a.isotropic_values is not None
    assert (a.c_A, a.C_A) == (1.0, 50.0) or abs(a.C_A - 50.0) < 1e-12


def test_non_spd_rejected_with_location():
    spec = GridSpec((1.0, 1.0), (3, 3))
    vals = np.ones((3, 3))
    vals[1, 2] = -1.0
    with pytest.raises(MaterialDataError, match="grid slot"):
        CoefficientField.isotropic(spec, vals)


def test_voxel_round_trip(tmp_path, rng):
    spec = GridSpec((1.0, 2.0), (5, 7))
    a = CoefficientField(spec, random_spd_packed(spec.shape, rng))
    save_coefficients(tmp_path / "a", a)
    b = load_voxel(tmp_path / "a.json")
    assert np.array_equal(a.components, b.components)
    u = GridField(spec, rng.standard_normal((2, 5, 7)))
    save_field(tmp_path / "u", u)
    assert np.array_equal(load_field(tmp_path / "u").values, u.values)
    (tmp_path / "bad.json").write_text('{"dim": 2, "shape": [4, 5], "half_periods": [1, 1], '
                                       '"kind": "isotropic", "dtype": "f64le", "order": "row-major-shifted"}')
    with pytest.raises(VoxelFormatError):
        load_voxel(tmp_path / "bad.json")


def test_chunked_bounds_equal_single_pass(rng, monkeypatch):
    spec = GridSpec((1.0,) * 3, (5, 7, 9))
    packed = random_spd_packed(spec.shape, rng)
    a = CoefficientField(spec, packed)
    monkeypatch.setattr(material, "_CHUNK", 17)
    b = CoefficientField(spec, packed)
    assert (a.c_A, a.C_A) == (b.c_A, b.C_A)


def _header_symbols():
    text = (ROOT / "include" / "fftcell_b200.h").read_text()
    return sorted(set(re.findall(r"\b(fc_[A-Za-z_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    bound = {name for name, _, _ in _native.SIGNATURES}
    assert set(syms) == bound


def test_no_gpu_fails_loudly():
    if _native.device_count() > 0:
        pytest.skip("a GPU is present")
    spec = GridSpec((1.0, 1.0), (5, 5))
    with pytest.raises(RuntimeError):
        _native.Context(spec)


def test_product_never_imports_oracle():
    for p in (ROOT / "paper_1311_0089_b200").rglob("*.py"):
        for line in p.read_text().splitlines():
            if line.strip().startswith(("import", "from")):
                assert "oracle" not in line, f"{p}: {line}"


@pytest.mark.parametrize("shape", [(81, 81), (27, 27, 27), (5,), (45, 45, 135), (255,), (243, 243, 243)])
def test_fixed_point_scale_is_the_reference_sum(shape):
    """solver._fp_scale == max(l2_norm(E_N), tiny) of the expanded constant field
    (solver.py:258) bit for bit, via the run-length pairwise sum that needs no
    expanded field (grids beyond host memory, e.g. 1215^3)."""
    from paper_1311_0089_b200.solver import _fp_scale
    from paper_1311_0089_b200.transforms import GridField, l2_norm

    spec = GridSpec((1.0,) * len(shape), shape)
    for seed in range(3):
        E = np.random.default_rng(seed).standard_normal(len(shape))
        assert _fp_scale(spec, E) == max(l2_norm(GridField.constant(spec, E)), np.finfo(float).tiny)


def test_pairwise_sum_runs_matches_numpy(rng):
    from paper_1311_0089_b200.transforms import pairwise_sum_runs

    for counts in ([1], [7, 3], [128, 129], [1000, 1, 5000], [8191, 8193, 3]):
        vals = rng.standard_normal(len(counts))
        assert pairwise_sum_runs(vals, counts) == np.sum(np.repeat(vals, counts))


def test_from_phases_is_the_gathered_field(rng):
    """CoefficientField.from_phases: host-side the field is exactly what from_matrices
    builds from the gathered tensors (material.py:135-145); the phase form rides along
    for the device upload (uint16 labels + (nsym, n_phases) table)."""
    spec = GridSpec((1.0, 2.0, 0.5), (5, 7, 3))
    q = rng.standard_normal((4, 3, 3))
    tensors = q @ np.swapaxes(q, 1, 2) + 0.5 * np.eye(3)
    labels = rng.integers(0, 4, size=spec.shape)
    a = CoefficientField.from_phases(spec, labels, tensors)
    b = CoefficientField.from_matrices(spec, np.moveaxis(tensors[labels], (-2, -1), (0, 1)))
    assert np.array_equal(a.components, b.components)
    assert (a.c_A, a.C_A) == (b.c_A, b.C_A)
    lab16, table = a.phases
    assert lab16.dtype == np.uint16 and lab16.shape == spec.shape and table.shape == (6, 4)
    assert np.array_equal(table[:, lab16], a.components)
    assert b.phases is None
    # isotropic phases stay on the scalar path; d = 1 has no packed kernels
    iso = CoefficientField.from_phases(spec, labels, np.array([k + 1.0 for k in range(4)])[:, None, None] * np.eye(3))
    assert iso.phases is None and iso.isotropic_values is not None
    with pytest.raises(MaterialDataError):
        CoefficientField.from_phases(spec, labels, tensors[:3])  # label 3 out of range
    with pytest.raises(MaterialDataError):
        CoefficientField.from_phases(spec, labels[:-1], tensors)
    bad = tensors.copy()
    bad[0, 0, 1] += 1.0
    with pytest.raises(MaterialDataError):
        CoefficientField.from_phases(spec, labels, bad)
