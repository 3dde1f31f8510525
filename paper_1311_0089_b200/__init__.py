"""B200-native GaNi cell-problem solver (arXiv 1311.0089), reference-shaped API.

Mirrors the solver path of the reference package ``fftcell``: grid and
material setup, ``solve_cg`` / ``solve_neumann`` (alias ``fixed_point``),
``solve``, ``apply_system``, ``residual_norm`` and ``effective_tensor``.
All numerics run in hand-written sm_100a CUDA (``csrc/``) behind the C ABI of
``include/fftcell_b200.h``; there is no CPU fallback.
"""

from .grid import GridSpec, frequency, grid_point, iter_lattice
from .green import ReferenceTensor
from .material import (
    CoefficientField,
    MaterialDataError,
    VoxelFormatError,
    apply_A,
    load_field,
    load_voxel,
    sample_analytic,
    save_coefficients,
    save_field,
)
from .transforms import GridField, l2_inner, l2_norm
from .solver import (
    LoadCase,
    SolveReport,
    SolverConfig,
    apply_system,
    default_reference,
    residual_norm,
    solve,
    solve_batch,
    solve_cg,
    solve_fixed_point,
    solve_neumann,
)
from .homogenize import ConvergenceError, EffectiveTensor, effective_tensor, flux_field, mean_flux

__all__ = [
    "GridSpec", "GridField", "ReferenceTensor", "CoefficientField", "MaterialDataError",
    "VoxelFormatError", "LoadCase", "SolverConfig", "SolveReport", "EffectiveTensor",
    "ConvergenceError", "frequency", "grid_point", "iter_lattice", "apply_A", "sample_analytic",
    "load_voxel", "load_field", "save_coefficients", "save_field", "l2_inner", "l2_norm",
    "solve_cg", "solve_neumann", "solve_fixed_point", "solve", "solve_batch", "apply_system",
    "residual_norm", "default_reference", "effective_tensor", "flux_field", "mean_flux",
]
