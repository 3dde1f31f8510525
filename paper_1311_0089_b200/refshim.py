"""Drop-in shim: route the reference package's hot path through the B200 library.

The reference (``fftcell``) has no FFI; its boundary is the Python call
signature of ``fftcell.solver``.  ``install()`` replaces, in
the imported reference package, exactly the hot-path entry points --

* ``solver.solve_cg`` / ``solve_neumann`` / ``solve`` / ``apply_system``
  (``solver.py:125-129,142-230,238-301``) and ``solver._Projector``
  (``solver.py:90-122``),
* and the copies its callers bound at import: ``homogenize.solve``
  (``homogenize.py:21``), ``analysis.solve_cg`` / ``solve_neumann`` /
  ``_Projector`` (``analysis.py:18``), ``cli.solve`` (``cli.py:38``)

-- with wrappers that take and return the REFERENCE's own types
(``CoefficientField``, ``LoadCase``, ``SolverConfig``, ``GridField``,
``SolveReport``) and compute on the GPU through this package (C ABI,
``include/fftcell_b200.h``).  Validation and messages are the reference's:
configs are re-validated by the reference's ``SolverConfig.__post_init__``,
non-convergence is a report, not an exception.  Everything else of the
reference (grids, materials, families, analysis, CLI plumbing, CSV writers)
stays untouched.  ``residual_norm`` and ``effective_tensor`` route through the
patched module globals.

Used by the pytest plugin ``paper_1311_0089_b200.refshim_pytest`` to run the
reference's own test suite against the GPU path (tools/run_reference_suite.sh).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .grid import GridSpec
from .green import ReferenceTensor
from .material import CoefficientField
from .solver import LoadCase, SolverConfig
from .solver import solve_cg as _solve_cg
from .solver import solve_neumann as _solve_neumann

CALLS = {"solve_cg": 0, "solve_neumann": 0, "apply_system": 0, "projector": 0}


def _spec(ref_spec):
    return GridSpec(tuple(ref_spec.half_periods), tuple(ref_spec.shape))


def _field(a):
    """The reference CoefficientField as ours, uploaded once (cached on the object)."""
    f = a.__dict__.get("_b200")
    if f is None:
        f = CoefficientField(_spec(a.spec), np.asarray(a.components, dtype=float))
        object.__setattr__(a, "_b200", f)
    return f


def _ref_tensor(ref):
    if ref is None:
        return None
    return ReferenceTensor(np.asarray(ref.matrix, dtype=float), ref.scalar_mode)


def install(fftcell=None):
    """Patch the imported reference package (``import fftcell`` if not given)."""
    if fftcell is None:
        import fftcell  # noqa: F401  (the reference, from PYTHONPATH)
    import fftcell.analysis as RA
    import fftcell.cli as RC
    import fftcell.homogenize as RH
    import fftcell.solver as RS

    def report(rep, ref_spec, method):
        sol = RS.GridField(ref_spec, rep.solution.values)
        its = tuple(RS.GridField(ref_spec, it.values) for it in rep.iterates)
        return RS.SolveReport(sol, rep.iterations, tuple(rep.residual_history), rep.converged, method,
                              rep.message, its)

    def solve_cg(a, load, cfg, init=None, record_iterates=False):
        """solver.py:142-230 on the GPU."""
        if cfg.method != "cg":
            raise ValueError("config method is not 'cg'")
        if len(load.E) != a.spec.dim:
            raise ValueError("load case dimension does not match grid")
        CALLS["solve_cg"] += 1
        ours = SolverConfig("cg", cfg.tol, cfg.max_iter, _ref_tensor(cfg.reference))
        init_vals = None if init is None else np.asarray(init.values, dtype=float)
        rep = _solve_cg(_field(a), LoadCase(load.E), ours, init=init_vals, record_iterates=record_iterates)
        return report(rep, a.spec, "cg")

    def solve_neumann(a, load, cfg):
        """solver.py:238-295 on the GPU; the default reference from the
        reference field's own bounds (solver.py:233-235)."""
        if len(load.E) != a.spec.dim:
            raise ValueError("load case dimension does not match grid")
        CALLS["solve_neumann"] += 1
        ref = cfg.reference if cfg.reference is not None else RS.default_reference(a)
        ours = SolverConfig("neumann", cfg.tol, cfg.max_iter, _ref_tensor(ref))
        rep = _solve_neumann(_field(a), LoadCase(load.E), ours)
        return report(rep, a.spec, "neumann")

    def solve(a, load, cfg, init=None):
        """solver.py:298-301."""
        if cfg.method == "cg":
            return solve_cg(a, load, cfg, init=init)
        return solve_neumann(a, load, cfg)

    def apply_system(a, u):
        """solver.py:125-129: G A u."""
        if a.spec != u.spec:
            raise ValueError("coefficient field and grid field specs do not match")
        CALLS["apply_system"] += 1
        return RS.GridField(a.spec, _field(a).device().apply_system(np.asarray(u.values, dtype=float)))

    class _Projector:
        """solver.py:90-122 on the GPU (projections of (d, *N) arrays)."""

        def __init__(self, spec, ref=None):
            if ref is not None and ref.dim != spec.dim:
                raise ValueError(f"reference tensor dimension {ref.dim} does not match grid dimension {spec.dim}")
            self.spec = spec
            self.ref = ref
            self._ctx = _native.context_for_spec(_spec(spec))

        def apply_orthogonal(self, values):
            CALLS["projector"] += 1
            return self._ctx.project(0, None, np.asarray(values, dtype=float))

        def apply_gamma_ref(self, values):
            CALLS["projector"] += 1
            return self._ctx.project(1, np.asarray(self.ref.matrix, dtype=float), np.asarray(values, dtype=float))

    RS.solve_cg, RS.solve_neumann, RS.solve, RS.apply_system, RS._Projector = (
        solve_cg, solve_neumann, solve, apply_system, _Projector)
    RH.solve = solve
    RA.solve_cg, RA.solve_neumann, RA._Projector = solve_cg, solve_neumann, _Projector
    RC.solve = solve
    return CALLS
