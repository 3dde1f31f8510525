"""Matrix-free GaNi solvers on the GPU, with the reference's API.

Mirror of ``fftcell.solver`` (``/root/reference/pkg/src/fftcell/solver.py``):
the dataclasses, validation, messages and stopping rules are the reference's;
every operator application, inner product and vector update runs in the CUDA
library (``csrc/``) through the C ABI of ``include/fftcell_b200.h``:

* ``solve_cg``       -> ``fc_solve_cg``          (solver.py:142-230)
* ``solve_neumann``  -> ``fc_solve_fixed_point`` (solver.py:238-295)
* ``apply_system``   -> ``fc_apply_system``      (solver.py:125-129)
* ``_Projector``     -> ``fc_project``           (solver.py:90-122)

``SolverConfig(method="fixed_point")`` is accepted as an alias of the
reference's ``"neumann"`` (BASELINE north_star naming).  ``solve_batch``
solves several load cases in one batched device solve (independent alpha,
beta and stopping per load case, identical per-case arithmetic).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .green import ReferenceTensor
from .grid import GridSpec
from .material import CoefficientField, apply_A  # noqa: F401  (re-export like the reference)
from .transforms import GridField, l2_norm, pairwise_sum_runs

_DIVERGENCE_WINDOW = 10  # solver.py:27 (the device loop uses the same window)
_METHOD_ALIASES = {"cg": "cg", "neumann": "neumann", "fixed_point": "neumann"}


@dataclass(frozen=True)
class LoadCase:
    """Mean applied gradient E (``solver.py:30-50``)."""

    E: tuple

    def __post_init__(self):
        E = tuple(float(e) for e in self.E)
        if not all(np.isfinite(E)):
            raise ValueError(f"load case entries must be finite, got {E}")
        object.__setattr__(self, "E", E)

    @property
    def dim(self):
        return len(self.E)

    def expand(self, spec: GridSpec) -> GridField:
        if len(self.E) != spec.dim:
            raise ValueError("load case dimension does not match grid")
        return GridField.constant(spec, self.E)


@dataclass(frozen=True)
class SolverConfig:
    """``solver.py:53-74``; ``method`` in {"cg", "neumann", "fixed_point"}."""

    method: str = "cg"
    tol: float = 1e-6
    max_iter: int = 1000
    reference: ReferenceTensor | None = None

    def __post_init__(self):
        if self.method not in _METHOD_ALIASES:
            raise ValueError(f"unknown method {self.method!r}")
        object.__setattr__(self, "method", _METHOD_ALIASES[self.method])
        if not (0 < self.tol < 1):
            raise ValueError(f"tol must lie in (0, 1), got {self.tol}")
        if self.max_iter < 1:
            raise ValueError("max_iter must be positive")
        if self.method == "cg" and self.reference is not None and self.reference.scalar_mode is None:
            raise ValueError("the CG route requires a scalar reference (lambda * I)")


@dataclass(frozen=True)
class SolveReport:
    """``solver.py:77-87``."""

    solution: GridField
    iterations: int
    residual_history: tuple
    converged: bool
    method: str
    message: str = ""
    iterates: tuple = ()


class _Projector:
    """Device Fourier projectors for one (spec, reference) pair (``solver.py:90-122``).

    Nothing spectral is stored: the GPU recomputes xi(k) from the slot index.
    """

    def __init__(self, spec: GridSpec, ref: ReferenceTensor | None = None):
        if ref is not None and ref.dim != spec.dim:  # the reference's einsum raises here (solver.py:101-104)
            raise ValueError(f"reference tensor dimension {ref.dim} does not match grid dimension {spec.dim}")
        self.spec = spec
        self.ref = ref
        self._ctx = _native.context_for_spec(spec)

    def apply_orthogonal(self, values):
        return self._ctx.project(0, None, values)

    def apply_gamma_ref(self, values):
        if self.ref is None:
            raise ValueError("apply_gamma_ref needs a reference tensor")
        return self._ctx.project(1, self.ref.matrix, values)


def apply_system(a: CoefficientField, u: GridField) -> GridField:
    """``G A u`` with the orthogonal G (``solver.py:125-129``)."""
    if a.spec != u.spec:
        raise ValueError("coefficient field and grid field specs do not match")
    return GridField(a.spec, a.device().apply_system(u.values))


def residual_norm(a: CoefficientField, load: LoadCase, candidate: GridField) -> float:
    """``|G A (candidate + E_N)|`` (``solver.py:132-135``)."""
    total = GridField(a.spec, candidate.values + load.expand(a.spec).values)
    return l2_norm(apply_system(a, total))


def _loads_array(loads, spec):
    for ld in loads:
        if len(ld.E) != spec.dim:
            raise ValueError("load case dimension does not match grid")
    return np.array([ld.E for ld in loads], dtype=float)


def _cg_reports(a, loads, cfg, init=None, record_iterates=False, want_solution=True):
    if cfg.method != "cg":
        raise ValueError("config method is not 'cg'")
    spec = a.spec
    if cfg.reference is not None and cfg.reference.dim != spec.dim:  # solver.py:161 builds _Projector(spec, ref)
        raise ValueError(f"reference tensor dimension {cfg.reference.dim} does not match grid dimension {spec.dim}")
    E = _loads_array(loads, spec)
    lam = None if cfg.reference is None else cfg.reference.scalar_mode
    init_vals = None
    if init is not None:
        init_vals = np.asarray(init.values if isinstance(init, GridField) else init, dtype=float)
    outs, x, its = a.device().solve_cg(E, cfg.tol, cfg.max_iter, lam=lam, init=init_vals,
                                       want_x=want_solution, record_iterates=record_iterates)
    reports = []
    for r, o in enumerate(outs):
        msg = ""
        if o["status"] == _native.ST_BREAKDOWN:
            msg = f"operator lost positive definiteness (pAp={o['detail']:.3e})"
        iterates = ()
        if its is not None:
            iterates = tuple(GridField(spec, its[k, r]) for k in range(min(len(its), o["iterations"] + 1)))
        sol = GridField(spec, x[r]) if x is not None else None
        reports.append(SolveReport(sol, o["iterations"], tuple(float(h) for h in o["history"]),
                                   o["converged"], "cg", message=msg, iterates=iterates))
    return reports


def solve_cg(a: CoefficientField, load: LoadCase, cfg: SolverConfig, init: GridField | None = None,
             record_iterates: bool = False) -> SolveReport:
    """Projected CG on ``G A e~ = -G A E`` (``solver.py:142-230``)."""
    return _cg_reports(a, [load], cfg, init=init, record_iterates=record_iterates)[0]


def default_reference(a: CoefficientField) -> ReferenceTensor:
    """``A0 = (c_A + C_A)/2 * I`` (``solver.py:233-235``)."""
    return ReferenceTensor.scalar(0.5 * (a.c_A + a.C_A), a.spec.dim)


def _fp_scale(spec, E):
    """``max(l2_norm(E_N), tiny)`` (``solver.py:258``): the reference's
    ``np.sum(E_N * E_N) / |N|`` reproduced bit for bit on any grid without
    expanding E_N (transforms.pairwise_sum_runs)."""
    E = np.asarray(E, dtype=float)
    s = pairwise_sum_runs(E * E, [spec.total] * spec.dim)
    val = float(np.sqrt(max(float(s / spec.total), 0.0)))
    return max(val, np.finfo(float).tiny)


def _fp_reports(a, loads, cfg, want_solution=True):
    ref = cfg.reference if cfg.reference is not None else default_reference(a)
    if ref.dim != a.spec.dim:
        raise ValueError("reference tensor dimension does not match grid")
    spec = a.spec
    E = _loads_array(loads, spec)
    scale = [_fp_scale(spec, e) for e in E]
    outs, x = a.device().solve_fixed_point(E, cfg.tol, cfg.max_iter, ref.matrix, scale, want_x=want_solution)
    reports = []
    for r, o in enumerate(outs):
        msg = ""
        if o["status"] == _native.ST_DIVERGENT:
            msg = f"divergent fixed-point iteration for reference tensor {ref.matrix.tolist()}"
        sol = GridField(spec, x[r]) if x is not None else None
        reports.append(SolveReport(sol, o["iterations"], tuple(float(h) for h in o["history"]),
                                   o["converged"], "neumann", message=msg))
    return reports


def solve_neumann(a: CoefficientField, load: LoadCase, cfg: SolverConfig) -> SolveReport:
    """Fixed point ``e <- E - Gamma0 (A - A0) e`` (``solver.py:238-295``)."""
    return _fp_reports(a, [load], cfg)[0]


solve_fixed_point = solve_neumann


def solve(a: CoefficientField, load: LoadCase, cfg: SolverConfig, init=None):
    """Dispatch by method (``solver.py:298-301``)."""
    if cfg.method == "cg":
        return solve_cg(a, load, cfg, init=init)
    return solve_neumann(a, load, cfg)


def solve_batch(a: CoefficientField, loads, cfg: SolverConfig, want_solution: bool = True):
    """Solve several load cases in one batched device solve (at most 8 per call)."""
    loads = list(loads)
    out = []
    for s in range(0, len(loads), _native.MAX_RHS):
        chunk = loads[s:s + _native.MAX_RHS]
        if cfg.method == "cg":
            out += _cg_reports(a, chunk, cfg, want_solution=want_solution)
        else:
            out += _fp_reports(a, chunk, cfg, want_solution=want_solution)
    return out
