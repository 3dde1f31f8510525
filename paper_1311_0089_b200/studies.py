"""Contrast and convergence studies on the GPU solver.

Counterpart of ``fftcell.analysis.contrast_study`` / ``convergence_study``
(``analysis.py:113-181``) with the solves on the device, so the studies run at
grid sizes where the CPU reference is impractical (e.g. the cfg2 medium at
2187^2 over four decades of contrast).  Media come from a callable instead of
the reference's analytic ``Family`` objects (``families.py``, out of scope):
``make_field(rho)`` for the contrast study, ``make_field(shape)`` for the
convergence study; ``checkerboard_2d`` and the BASELINE generators
(``generators.py``) are ready-made makers.

The fitted quantity and its rules follow the reference: least-squares slope of
log(values) against log(axis), with the first point dropped while that raises
R^2 by more than 0.05 (``analysis.py:46-70``); non-converged points are
recorded at their iteration count and flagged ``censored:<rho>``
(``analysis.py:151-181``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import GridSpec, axis_indices
from .material import CoefficientField
from .solver import LoadCase, SolverConfig, solve_cg, solve_neumann

R2_DROP = 0.05  # analysis.py:21


@dataclass(frozen=True)
class StudyResult:
    """Axis, values and the log-log fit of a rate claim (``analysis.py:27-43``)."""

    axis: tuple
    values: tuple
    fitted_exponent: float
    fit_quality: float
    label: str = ""
    flags: tuple = ()

    def __post_init__(self):
        axis = tuple(float(a) for a in self.axis)
        steps = np.diff(axis)
        if len(axis) > 1 and not (np.all(steps > 0) or np.all(steps < 0)):
            raise ValueError("study axis must be strictly monotone")
        object.__setattr__(self, "axis", axis)
        object.__setattr__(self, "values", tuple(float(v) for v in self.values))


def fit_loglog(axis, values):
    """(slope, R^2) of log(values) vs log(axis), pre-asymptotic points dropped."""
    lx = np.log(np.asarray(axis, dtype=float))
    ly = np.log(np.asarray(values, dtype=float))

    def line(xs, ys):
        slope, icept = np.polyfit(xs, ys, 1)
        resid = float(np.sum((ys - (slope * xs + icept)) ** 2))
        spread = float(np.sum((ys - ys.mean()) ** 2))
        return float(slope), (1.0 if spread == 0 else 1.0 - resid / spread)

    slope, r2 = line(lx, ly)
    while len(lx) > 3:
        s2, q2 = line(lx[1:], ly[1:])
        if q2 - r2 <= R2_DROP:
            break
        lx, ly, slope, r2 = lx[1:], ly[1:], s2, q2
    return slope, r2


def _result(axis, values, label, flags=()):
    if len(values) >= 2 and all(v > 0 for v in values):
        k, q = fit_loglog(axis, values)
    else:
        k, q = float("nan"), float("nan")
        flags = tuple(flags) + ("no-fit",)
    return StudyResult(tuple(axis), tuple(values), k, q, label, tuple(flags))


def checkerboard_2d(shape, a1, a2, half_periods=(1.0, 1.0)):
    """Quadrant checkerboard on the cell (``families.py:109-138``), sampled at the
    grid points x = k h: a1 where x0 x1 > 0, a2 where x0 x1 < 0 and sqrt(a1 a2)
    on the interface lines (odd grids sample x = 0 exactly)."""
    spec = GridSpec(tuple(half_periods), tuple(shape))
    s0 = np.sign(axis_indices(spec.shape[0]))[:, None]
    s1 = np.sign(axis_indices(spec.shape[1]))[None, :]
    s = s0 * s1
    vals = np.where(s > 0, float(a1), np.where(s < 0, float(a2), float(np.sqrt(a1 * a2))))
    return CoefficientField.isotropic(spec, vals)


def contrast_study(make_field, contrasts, tol=1e-6, max_iter=100000, methods=("cg", "neumann"), load=None):
    """Iterations to tolerance vs coefficient contrast, per method (``analysis.py:151-181``).

    ``make_field(rho)`` returns the CoefficientField at contrast rho; the fixed
    point uses the default reference ((c_A + C_A) / 2) I.  Returns
    ``{method: StudyResult}`` plus ``"reports"``: the per-contrast SolveReports."""
    contrasts = list(contrasts)
    fields = {rho: make_field(rho) for rho in contrasts}
    out = {"reports": {}}
    for method in methods:
        its, flags, reps = [], [], []
        for rho in contrasts:
            a = fields[rho]
            ld = load or LoadCase(tuple(np.eye(a.spec.dim)[0]))
            cfg = SolverConfig(method=method, tol=tol, max_iter=max_iter)
            rep = solve_cg(a, ld, cfg) if method == "cg" else solve_neumann(a, ld, cfg)
            reps.append(rep)
            its.append(max(rep.iterations, 1))
            if not rep.converged:
                flags.append(f"censored:{rho:g}")
        out[method] = _result(contrasts, its, f"contrast:{method}", flags)
        out["reports"][method] = tuple(reps)
    return out


def _prolong(coarse_hat, fine_shape):
    """Zero-pad coarse DFT coefficients (storage order) onto a finer lattice
    (``analysis.py:80-92``)."""
    d = coarse_hat.shape[0]
    out = np.zeros((d,) + tuple(fine_shape), dtype=complex)
    slots = [np.fft.fftfreq(nc, d=1.0 / nc).round().astype(int) % nf
             for nc, nf in zip(coarse_hat.shape[1:], fine_shape)]
    out[np.ix_(np.arange(d), *slots)] = coarse_hat
    return out


def spectral_error(coarse, fine):
    """L2 distance of two trigonometric polynomials on nested grids
    (``analysis.py:95-99``; DFT with 1/|N| on the forward transform)."""
    axes_c = tuple(range(1, coarse.ndim))
    c = np.fft.fftn(coarse, axes=axes_c) / np.prod(coarse.shape[1:])
    f = np.fft.fftn(fine, axes=axes_c) / np.prod(fine.shape[1:])
    return float(np.sqrt(np.sum(np.abs(_prolong(c, fine.shape[1:]) - f) ** 2)))


def convergence_study(make_field, grids, cfg, load=None, ref_factor=4, regularity="low-regularity"):
    """Solution error vs the largest grid spacing over a sequence of odd grids
    (``analysis.py:113-148``): the reference solution is computed on a
    ``ref_factor`` x finer grid (n -> ref_factor n + 1) and errors are measured
    after spectral prolongation.  ``make_field(shape)`` samples the medium."""
    grids = [tuple(g) for g in grids]
    ref_shape = tuple(ref_factor * n + 1 for n in grids[-1])
    ref_a = make_field(ref_shape)
    ld = load or LoadCase(tuple(np.eye(ref_a.spec.dim)[0]))
    ref = solve_cg(ref_a, ld, cfg)
    if not ref.converged:
        raise RuntimeError("reference solve did not converge")
    axis, values = [], []
    for shape in grids:
        a = make_field(shape)
        rep = solve_cg(a, ld, cfg)
        if not rep.converged:
            raise RuntimeError(f"study solve on {shape} did not converge")
        axis.append(max(a.spec.spacings))
        values.append(spectral_error(rep.solution.values, ref.solution.values))
    flags = () if regularity == "smooth" else ("low-regularity",)
    order = np.argsort(axis)[::-1]  # coarsest first (the drop rule removes pre-asymptotic points)
    axis = [axis[i] for i in order]
    values = [values[i] for i in order]
    if all(v > 0 for v in values) and any(b > a for a, b in zip(values[:-1], values[1:])):
        flags = flags + ("non-monotone",)
    return _result(axis, values, f"convergence:{getattr(make_field, '__name__', 'field')}", flags)
