"""Slab decomposition checked on ONE GPU: P slabs of the same
device emulate P ranks (no kernel ever waits on another).  Every result must
match the single-slab run: identical iteration counts, fields to rounding."""

import numpy as np
import pytest

from conftest import random_spd_packed, rel_l2
from paper_1311_0089_b200 import _native, generators as gen
from paper_1311_0089_b200.grid import GridSpec

pytestmark = pytest.mark.gpu


def _pair(spec, packed=None, iso=None, P=2):
    one = _native.Context(spec)
    many = _native.Context(spec, slabs=[0] * P)
    for ctx in (one, many):
        if iso is not None:
            lib_kind, host = 0, np.ascontiguousarray(iso)
        else:
            lib_kind, host = 1, np.ascontiguousarray(packed)
        _native._check(_native.lib().fc_set_coefficients(ctx._h, lib_kind, _native._ptr(host), host.size))
    return one, many


@pytest.mark.parametrize("P", [2, 3, 4])
def test_sharded_operators_match_single(P, rng):
    spec = GridSpec((1.0, 1.5, 0.75), (27, 9, 81))
    packed = random_spd_packed(spec.shape, rng)
    one, many = _pair(spec, packed=packed, P=P)
    u = rng.standard_normal((2, 3) + spec.shape)
    for f in ("apply_system", "apply_A"):
        a, b = getattr(one, f)(u), getattr(many, f)(u)
        assert np.max(np.abs(a - b)) <= 1e-13 * np.max(np.abs(a))
    A0 = np.array([[2.0, 0.3, 0.0], [0.3, 1.5, 0.1], [0.0, 0.1, 1.0]])
    for which, ref in ((0, None), (1, A0)):
        a, b = one.project(which, ref, u), many.project(which, ref, u)
        assert np.max(np.abs(a - b)) <= 1e-13 * max(1.0, np.max(np.abs(a)))


@pytest.mark.parametrize("P", [2, 3, 5])
def test_sharded_cg_fixed_point_energy(P):
    a = gen.cfg3_sphere(27)
    one, many = _pair(a.spec, iso=a.isotropic_values, P=P)
    E = np.array([[1.0, 0.0, 0.0], [0.2, -0.5, 1.0]])
    r1, x1, _ = one.solve_cg(E, 1e-8, 500)
    rP, xP, _ = many.solve_cg(E, 1e-8, 500)
    for q1, qP in zip(r1, rP):
        assert q1["iterations"] == qP["iterations"] and qP["converged"]
        np.testing.assert_allclose(qP["history"], q1["history"], rtol=1e-9, atol=1e-12 * q1["history"][0])
    assert rel_l2(xP, x1) <= 1e-12
    np.testing.assert_allclose(many.energy(E), one.energy(E), rtol=1e-13)
    lam = 0.5 * (1.0 + 50.0)
    f1, e1 = one.solve_fixed_point(E[:1], 1e-6, 1000, lam * np.eye(3), [1.0])
    fP, eP = many.solve_fixed_point(E[:1], 1e-6, 1000, lam * np.eye(3), [1.0])
    assert f1[0]["iterations"] == fP[0]["iterations"] and fP[0]["converged"]
    assert rel_l2(eP, e1) <= 1e-12


def test_sharded_polycrystal_device_generator_and_warm_start():
    n = 27
    spec = GridSpec((1.0,) * 3, (n,) * 3)
    seeds, packed = gen.cfg4_grains(512, gen.SEEDS["cfg4"], n)
    one = _native.Context(spec)
    many = _native.Context(spec, slabs=[0, 0, 0])
    for ctx in (one, many):
        ctx.generate_voronoi(seeds, packed)
    E = np.array([[1.0, 0.0, 0.0]])
    r1, x1, _ = one.solve_cg(E, 1e-8, 2000)
    rP, xP, _ = many.solve_cg(E, 1e-8, 2000)
    assert r1[0]["iterations"] == rP[0]["iterations"]
    # this 27^3 / 512-grain case amplifies rounding: two runs of the unmodified reference
    # differ by 1.45e-9 (tests/golden/poly27.npz cg_floor); gate at 10x that floor
    assert rel_l2(xP, x1) <= 1.5e-8
    w1, _, _ = one.solve_cg(E, 1e-8, 2000, init=x1)
    wP, _, _ = many.solve_cg(E, 1e-8, 2000, init=x1)
    assert w1[0]["iterations"] == wP[0]["iterations"] <= 2


def test_nccl_slab_path_single_rank():
    """fc_create_dist with one rank: the NCCL exchange (send/recv to self) and the
    all-gather reduction run for real and must reproduce the plain context."""
    import torch  # noqa: F401  (loads the NCCL the library resolves at run time)

    a = gen.cfg3_sphere(27)
    one = _native.Context(a.spec)
    dist = _native.Context.distributed(a.spec, 1, 0, 0, _native.nccl_unique_id())
    for ctx in (one, dist):
        ctx.set_coefficients(a)
    E = np.array([[1.0, 0.0, 0.0]])
    r1, x1, _ = one.solve_cg(E, 1e-8, 500)
    rD, xD, _ = dist.solve_cg(E, 1e-8, 500)
    assert r1[0]["iterations"] == rD[0]["iterations"]
    assert rel_l2(xD, x1) <= 1e-13
    np.testing.assert_allclose(dist.energy(E), one.energy(E), rtol=1e-13)


@pytest.mark.parametrize("P", [2, 3])
def test_sharded_generic_lengths(P, rng):
    """Axes that are not powers of three (the cfg5 grid 1215 = 3^5 5 class) run
    the shared-memory Stockham kernels, which take the same slab maps: a 45 x 25
    x 15 grid on P slabs matches the single slab, and the single slab matches
    the CPU oracle."""
    import os

    from oracle import fftcell_oracle as orc

    shape = (45, 25, 15)
    spec = GridSpec((1.0, 1.0, 1.0), shape)
    a = np.where(rng.random(shape) < 0.3, 20.0, 1.0)
    one, many = _pair(spec, iso=a, P=P)
    u = rng.standard_normal((2, 3) + shape)
    s1, sP = one.apply_system(u), many.apply_system(u)
    assert np.max(np.abs(s1 - sP)) <= 1e-13 * np.max(np.abs(s1))
    E = np.array([[1.0, 0.0, 0.0], [0.0, 0.6, 0.8]])
    r1, x1, _ = one.solve_cg(E, 1e-8, 500)
    rP, xP, _ = many.solve_cg(E, 1e-8, 500)
    assert [q["iterations"] for q in r1] == [q["iterations"] for q in rP]
    assert rel_l2(xP, x1) <= 1e-12
    ref = orc.solve_cg(orc.isotropic_full(a, 3), tuple(E[0]), shape, (1.0, 1.0, 1.0), 1e-8, 500)
    assert r1[0]["iterations"] == ref["iterations"]
    assert rel_l2(x1[0], ref["solution"]) < 1e-9


def test_sharded_forced_generic_matches_register_path():
    """Plan option force_generic routes a power-of-three grid through the Stockham
    kernels; sharded over 3 slabs it must reproduce the register-path solve."""
    a = gen.cfg3_sphere(27)
    E = np.array([[1.0, 0.0, 0.0]])
    reg = _native.Context(a.spec)
    reg.set_coefficients(a)
    r0, x0, _ = reg.solve_cg(E, 1e-8, 500)
    with _native.plan_options(force_generic=1):
        gen_many = _native.Context(a.spec, slabs=[0, 0, 0])
    gen_many.set_coefficients(a)
    r1, x1, _ = gen_many.solve_cg(E, 1e-8, 500)
    assert r0[0]["iterations"] == r1[0]["iterations"]
    assert rel_l2(x1, x0) <= 1e-12


@pytest.mark.parametrize("P", [2, 4])
def test_fused_exchange_matches_copy_exchange(P):
    """Fused exchange (the sweeps store straight into the other slabs' buffers)
    against the copy-engine exchange: same arithmetic, bitwise-identical solve."""
    a = gen.cfg3_sphere(27)
    E = np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    fused = _native.Context(a.spec, slabs=[0] * P)
    fused.set_coefficients(a)
    rf, xf, _ = fused.solve_cg(E, 1e-8, 500)
    with _native.plan_options(fused_exchange=0):
        copy = _native.Context(a.spec, slabs=[0] * P)
    copy.set_coefficients(a)
    rc, xc, _ = copy.solve_cg(E, 1e-8, 500)
    assert [q["iterations"] for q in rf] == [q["iterations"] for q in rc]
    assert np.array_equal(xf, xc)
    u = np.random.default_rng(5).standard_normal((2, 3) + a.spec.shape)
    assert np.array_equal(fused.apply_system(u), copy.apply_system(u))


def test_cfg5_device_generator_matches_host():
    """fc_spheres_stamp / fc_spheres_finish (device cfg5) against the host
    generator at 81^3 (radius 20 x 81 / 1215): same centre count, and the CG
    solve on the device-built field equals the one on the uploaded host field
    bit for bit (same coefficients); also built across 3 slabs."""
    n = 81
    spec = GridSpec((1.0,) * 3, (n,) * 3)
    centres, covered = gen.cfg5_sphere_centres(n, gen.SEEDS["cfg5"], 20.0 * n / 1215.0)
    host = _native.Context(spec)
    host.set_coefficients(gen.cfg5_two_phase(n))
    dev = _native.Context(spec)
    used = gen.cfg5_device(dev, n)
    assert used.shape == centres.shape and np.array_equal(used, centres)
    E = np.array([gen.CFG5_LOAD])
    r0, x0, _ = host.solve_cg(E, 1e-8, 1000)
    r1, x1, _ = dev.solve_cg(E, 1e-8, 1000)
    assert r0[0]["iterations"] == r1[0]["iterations"]
    assert np.array_equal(x0, x1)
    many = _native.Context(spec, slabs=[0, 0, 0])
    gen.cfg5_device(many, n)
    r2, x2, _ = many.solve_cg(E, 1e-8, 1000)
    assert r2[0]["iterations"] == r0[0]["iterations"]
    assert rel_l2(x2, x0) <= 1e-12


@pytest.mark.parametrize("max_iter", [5, 500])
def test_sharded_deferred_x_update_is_bitwise_identical(max_iter):
    """Sharded CG with the x update deferred into the first sweep (default)
    equals the immediate update (plan option defer_x = 0) bit for bit,
    including the flush of RHSs stopped by max_iter."""
    a = gen.cfg3_sphere(27)
    E = np.array([[1.0, 0.0, 0.0], [0.2, -0.5, 1.0]])
    _, many = _pair(a.spec, iso=a.isotropic_values, P=3)
    r1, x1, _ = many.solve_cg(E, 1e-8, max_iter)
    with _native.plan_options(defer_x=0):
        _, imm = _pair(a.spec, iso=a.isotropic_values, P=3)
    r0, x0, _ = imm.solve_cg(E, 1e-8, max_iter)
    assert [q["iterations"] for q in r1] == [q["iterations"] for q in r0]
    assert np.array_equal(x1, x0), rel_l2(x1, x0)
