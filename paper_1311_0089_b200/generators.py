"""Seeded synthetic microstructures for the five BASELINE configurations.

The reference has no generator for these (its analytic families, ``families.py``,
sample through a per-point Python loop, ``material.py:161-179``, which is
unusable beyond ~10^6 voxels).  These are the generator contracts of
``SURVEY.md`` §8(d), vectorised with numpy so the oracle and the GPU path
consume the *same* arrays.  Positions follow the storage contract of
``grid.py:9-20,131-139``: slot ``i`` holds the centred index ``k`` and the
grid point ``x = k h`` with ``h = 2Y/N``.

Every config is on the cell ``[-1, 1]^d`` (half periods 1).
"""

from __future__ import annotations

import numpy as np

from .grid import GridSpec, axis_indices
from .material import CoefficientField

SEEDS = {"cfg2": 2187, "cfg4": 729, "cfg5": 1215}


def _coords(spec):
    """Per-axis grid-point coordinates ``k_a h_a`` in storage order."""
    return [axis_indices(n) * h for n, h in zip(spec.shape, spec.spacings)]


def cfg1_square_inclusion(n=81, inside=10.0, outside=1.0, side=0.6):
    """cfg1: centred square |x0|,|x1| < side on [-1,1]^2, A=10 inside, 1 outside."""
    spec = GridSpec((1.0, 1.0), (n, n))
    x0, x1 = np.meshgrid(*_coords(spec), indexing="ij")
    mask = (np.abs(x0) < side) & (np.abs(x1) < side)
    return CoefficientField.isotropic(spec, np.where(mask, inside, outside))


def cfg2_phase_mask(n=2187, seed=SEEDS["cfg2"], sigma=4.0, quantile=0.6):
    """cfg2 phase indicator: smoothed seeded white noise thresholded at its 0.6-quantile.

    White N(0,1) noise, periodic Gaussian filter (sigma in voxels) applied as the
    Fourier multiplier ``exp(-2 pi^2 sigma^2 (f0^2 + f1^2))``, ``f = fftfreq(n)``.
    """
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal((n, n))
    f = np.fft.fftfreq(n)
    mult = np.exp(-2.0 * np.pi**2 * sigma**2 * (f[:, None] ** 2 + f[None, :] ** 2))
    field = np.fft.ifft2(np.fft.fft2(noise) * mult).real
    return field > np.quantile(field, quantile)


def cfg2_random_two_phase(n=2187, seed=SEEDS["cfg2"], high=100.0, low=1.0):
    spec = GridSpec((1.0, 1.0), (n, n))
    return CoefficientField.isotropic(spec, np.where(cfg2_phase_mask(n, seed), high, low))


CFG2_LOADS = ((1.0, 0.0), (0.0, 1.0), (1.0 / np.sqrt(2.0), 1.0 / np.sqrt(2.0)))


def cfg3_sphere(n=243, inside=50.0, outside=1.0, radius=0.7):
    """cfg3: centred sphere |x|^2 < 0.7^2 (radius 0.35 x cell side 2)."""
    spec = GridSpec((1.0, 1.0, 1.0), (n, n, n))
    c = _coords(spec)
    r2 = c[0][:, None, None] ** 2 + c[1][None, :, None] ** 2 + c[2][None, None, :] ** 2
    return CoefficientField.isotropic(spec, np.where(r2 < radius**2, inside, outside))


def _haar_rotations(rng, m):
    """Haar-random rotations: QR of a Gaussian, columns sign-fixed by diag(R), det +1."""
    out = np.empty((m, 3, 3))
    for g in range(m):
        q, r = np.linalg.qr(rng.standard_normal((3, 3)))
        q = q * np.sign(np.diag(r))[None, :]
        if np.linalg.det(q) < 0:
            q[:, 0] = -q[:, 0]
        out[g] = q
    return out


def cfg4_grains(n_grains=512, seed=SEEDS["cfg4"], n=729):
    """cfg4 grain data: seed positions (voxel units on the torus [0,n)^3) and packed tensors.

    Per grain ``A_g = R diag(lambda) R^T`` with ``lambda_i = exp(N(0,1))`` and R Haar.
    Returns ``(seeds (G,3), packed (G,6))`` in the packed order of ``material.py:30-34``.
    """
    rng = np.random.default_rng(seed)
    seeds = rng.uniform(0.0, float(n), size=(n_grains, 3))
    lam = np.exp(rng.standard_normal((n_grains, 3)))
    rots = _haar_rotations(rng, n_grains)
    mats = np.einsum("gab,gb,gcb->gac", rots, lam, rots)
    mats = 0.5 * (mats + np.swapaxes(mats, 1, 2))
    packed = np.stack(
        [mats[:, 0, 0], mats[:, 1, 1], mats[:, 2, 2], mats[:, 0, 1], mats[:, 0, 2], mats[:, 1, 2]],
        axis=1,
    )
    return seeds, packed


def voronoi_labels(n, seeds, block=1 << 18):
    """Nearest seed (periodic minimum image, voxel centres at integer slots) per voxel.

    Squared distance is accumulated axis by axis in a fixed order so the device
    generator can reproduce the labels bit for bit.
    """
    idx = np.indices((n, n, n)).reshape(3, -1).T.astype(float)
    labels = np.empty(idx.shape[0], dtype=np.int32)
    for s in range(0, idx.shape[0], block):
        p = idx[s : s + block]
        best = np.full(p.shape[0], np.inf)
        lab = np.zeros(p.shape[0], dtype=np.int32)
        for g in range(seeds.shape[0]):
            d2 = np.zeros(p.shape[0])
            for a in range(3):
                t = np.abs(p[:, a] - seeds[g, a])
                t = np.minimum(t, n - t)
                d2 = d2 + t * t
            better = d2 < best
            best = np.where(better, d2, best)
            lab = np.where(better, g, lab)
        labels[s : s + block] = lab
    return labels.reshape(n, n, n)


def cfg4_polycrystal(n=729, n_grains=512, seed=SEEDS["cfg4"]):
    """cfg4 (host build; fine up to ~81^3, use the device generator beyond)."""
    seeds, packed = cfg4_grains(n_grains, seed, n)
    labels = voronoi_labels(n, seeds)
    spec = GridSpec((1.0, 1.0, 1.0), (n, n, n))
    return CoefficientField(spec, np.moveaxis(packed[labels], -1, 0).copy())


def cfg5_sphere_centres(n=1215, seed=SEEDS["cfg5"], radius=20.0, fraction=0.30, batch=64):
    """cfg5 inclusion centres: add seeded uniform centres until the periodic union of
    radius-``radius`` voxel balls covers ``fraction`` of the grid.

    Coverage is tracked exactly on the voxel grid, ``batch`` centres at a time; the
    returned list is truncated to the first centre at which coverage reaches the target.
    """
    rng = np.random.default_rng(seed)
    covered = np.zeros((n, n, n), dtype=bool)
    r = int(np.ceil(radius))
    off = np.arange(-r, r + 1)
    dz, dy, dx = np.meshgrid(off, off, off, indexing="ij")
    ball = (dz * dz + dy * dy + dx * dx) < radius * radius
    bz, by, bx = dz[ball], dy[ball], dx[ball]
    centres = []
    target = fraction * n**3
    count = 0
    while True:
        for c in rng.uniform(0.0, float(n), size=(batch, 3)):
            ci = np.floor(c).astype(np.int64)
            covered[(ci[0] + bz) % n, (ci[1] + by) % n, (ci[2] + bx) % n] = True
            centres.append(np.floor(c))
            count = int(covered.sum()) if len(centres) % 16 == 0 else count
            if len(centres) % 16 == 0 and count >= target:
                return np.array(centres), covered
        count = int(covered.sum())
        if count >= target:
            return np.array(centres), covered


def cfg5_two_phase(n=1215, seed=SEEDS["cfg5"], radius=None, high=1000.0, low=1.0):
    """cfg5 (host build for down-scaled instances; radius scales as 20 n / 1215)."""
    radius = 20.0 * n / 1215.0 if radius is None else radius
    _, covered = cfg5_sphere_centres(n, seed, radius)
    spec = GridSpec((1.0, 1.0, 1.0), (n, n, n))
    return CoefficientField.isotropic(spec, np.where(covered, high, low))


def cfg5_device(ctx, n=1215, seed=SEEDS["cfg5"], radius=None, fraction=0.30, high=1000.0, low=1.0, batch=64,
                count_fn=None):
    """cfg5 built on the device (fc_spheres_stamp): the same centre stream and
    stopping rule as ``cfg5_sphere_centres`` (coverage checked every 16 centres),
    so the field is bit-identical to ``cfg5_two_phase``.  ``count_fn`` sums the
    covered-voxel count over ranks (one slab per process); returns the centres used."""
    radius = 20.0 * n / 1215.0 if radius is None else radius
    rng = np.random.default_rng(seed)
    target = fraction * n**3
    used = []
    while True:
        cs = np.floor(rng.uniform(0.0, float(n), size=(batch, 3))).astype(np.int64)
        for g in range(0, batch, 16):
            grp = cs[g:g + 16]
            cov = ctx.spheres_stamp(grp, radius)
            if count_fn is not None:
                cov = count_fn(cov)
            used.append(grp)
            if cov >= target:
                ctx.spheres_finish(high, low)
                return np.concatenate(used).astype(np.float64)


CFG5_LOAD = (1.0 / np.sqrt(3.0),) * 3
