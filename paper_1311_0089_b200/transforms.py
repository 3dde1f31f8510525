"""Host containers and discrete mean inner product.

Mirror of the parts of ``fftcell.transforms`` the solver path uses
(``/root/reference/pkg/src/fftcell/transforms.py:37-61,168-180``).  The
``(d, *N)`` fp64 component-major layout of :class:`GridField` is exactly the
layout of the device vectors (one such block per right-hand side).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import GridSpec


@dataclass(frozen=True)
class GridField:
    """Real d-vector field, component-major ``(d, *N)`` (``transforms.py:37-61``)."""

    spec: GridSpec
    values: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.values, dtype=float)
        expected = (self.spec.dim,) + self.spec.shape
        if v.shape != expected:
            raise ValueError(f"values shape {v.shape} != expected {expected}")
        object.__setattr__(self, "values", v)

    @classmethod
    def zeros(cls, spec):
        return cls(spec, np.zeros((spec.dim,) + spec.shape))

    @classmethod
    def constant(cls, spec, vec):
        vec = np.asarray(vec, dtype=float)
        values = np.broadcast_to(
            vec.reshape((spec.dim,) + (1,) * spec.dim), (spec.dim,) + spec.shape
        ).copy()
        return cls(spec, values)


def l2_inner(u: GridField, v: GridField) -> float:
    """Discrete mean inner product ``(1/|N|) sum <u^k, v^k>`` (``transforms.py:168-176``)."""
    if u.spec != v.spec:
        raise ValueError("grid specs do not match")
    return float(np.sum(u.values * v.values) / u.spec.total)


def l2_norm(u: GridField) -> float:
    """``transforms.py:179-180``."""
    return float(np.sqrt(max(l2_inner(u, u), 0.0)))
