"""Voxel files straight into / out of HBM (the reference's
format, material.py:194-307): fc_load_coefficients / fc_save_solution stream the
payload through pinned staging buffers.  The device-loaded field must give the
same solve bits as the host-built field, its bounds must equal the host
closed-form bounds, and a streamed-out solution must read back identically."""

import numpy as np
import pytest

from conftest import random_spd_packed, rel_l2
from paper_1311_0089_b200 import (
    CoefficientField, GridSpec, LoadCase, SolverConfig, _native, generators as gen, solve_cg, solve_neumann,
)
from paper_1311_0089_b200.material import (
    MaterialDataError, VoxelFormatError, load_field, load_voxel, load_voxel_device, save_coefficients, save_voxel,
)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", ["iso3d", "packed3d", "packed2d"])
def test_device_loaded_field_solves_identically(tmp_path, case):
    rng = np.random.default_rng(3)
    if case == "iso3d":
        a = gen.cfg3_sphere(27)
        save_coefficients(tmp_path / "m", a, "isotropic")
        E = (1.0, 0.0, 0.0)
    elif case == "packed3d":
        spec = GridSpec((1.0, 1.0, 1.0), (27, 9, 81))
        a = CoefficientField(spec, random_spd_packed(spec.shape, rng))
        save_coefficients(tmp_path / "m", a)
        E = (0.2, 1.0, -0.5)
    else:
        spec = GridSpec((1.0, 1.5), (45, 33))
        a = CoefficientField(spec, random_spd_packed(spec.shape, rng))
        save_coefficients(tmp_path / "m", a)
        E = (1.0, 0.3)
    dev = load_voxel_device(tmp_path / "m.json")
    assert dev.spec == a.spec
    if case == "iso3d":
        assert (dev.c_A, dev.C_A) == (a.c_A, a.C_A)
    else:
        assert abs(dev.c_A - a.c_A) <= 1e-14 * a.C_A and abs(dev.C_A - a.C_A) <= 1e-14 * a.C_A
    cfg = SolverConfig(tol=1e-8, max_iter=2000)
    r0 = solve_cg(a, LoadCase(E), cfg)
    r1 = solve_cg(dev, LoadCase(E), cfg)
    assert r0.iterations == r1.iterations
    assert np.array_equal(r0.solution.values, r1.solution.values)
    # the solution streamed out of HBM reads back bit for bit
    dev.save_solution(tmp_path / "sol")
    back = load_field(tmp_path / "sol.json")
    assert np.array_equal(back.values, r1.solution.values)
    if case == "iso3d":  # default reference from the device bounds
        f0 = solve_neumann(a, LoadCase(E), SolverConfig(method="neumann", tol=1e-6, max_iter=2000))
        f1 = solve_neumann(dev, LoadCase(E), SolverConfig(method="neumann", tol=1e-6, max_iter=2000))
        assert f0.iterations == f1.iterations
        assert np.array_equal(f0.solution.values, f1.solution.values)


def test_sharded_context_loads_its_planes(tmp_path):
    a = gen.cfg3_sphere(27)
    save_coefficients(tmp_path / "m", a, "isotropic")
    E = np.array([[1.0, 0.0, 0.0]])
    one = _native.Context(a.spec)
    one.load_coefficients(tmp_path / "m.bin", 0)
    many = _native.Context(a.spec, slabs=[0, 0, 0])
    many.load_coefficients(tmp_path / "m.bin", 0)
    assert many.coefficient_bounds()[:2] == one.coefficient_bounds()[:2]
    r1, x1, _ = one.solve_cg(E, 1e-8, 500)
    rP, xP, _ = many.solve_cg(E, 1e-8, 500)
    assert r1[0]["iterations"] == rP[0]["iterations"]
    assert rel_l2(xP, x1) <= 1e-12
    many.save_solution(tmp_path / "x.bin")
    assert np.array_equal(np.fromfile(tmp_path / "x.bin", dtype="<f8").reshape(xP.shape), xP)


def test_device_load_errors(tmp_path):
    spec = GridSpec((1.0, 1.0), (9, 9))
    save_voxel(tmp_path / "m", spec, np.full(spec.shape, 2.0), "isotropic")
    with open(tmp_path / "m.bin", "ab") as fh:
        fh.write(b"\0" * 8)
    with pytest.raises(VoxelFormatError, match="expected"):
        load_voxel_device(tmp_path / "m.json")
    vals = np.full(spec.shape, 2.0)
    vals[3, 4] = -1.0
    save_voxel(tmp_path / "bad", spec, vals, "isotropic")
    with pytest.raises(MaterialDataError, match="grid slot"):
        load_voxel_device(tmp_path / "bad.json")
    with pytest.raises(MaterialDataError, match="grid slot"):
        load_voxel(tmp_path / "bad.json")
