"""Constant SPD reference tensor A0 (mirror of ``fftcell.green.ReferenceTensor``,
``/root/reference/pkg/src/fftcell/green.py:24-70``).

Only the tensor type lives on the host.  The Fourier multiplier
``Gamma_hat(k) = xi xi^T / <A0 xi, xi>`` (``green.py:73-92``) is evaluated on
the device inside the outer-axis FFT sweep, see ``csrc/fc_engine.cu``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ReferenceTensor:
    """Constant SPD reference tensor; ``scalar_mode`` set when A0 = lambda I."""

    matrix: np.ndarray
    scalar_mode: float | None = None

    def __post_init__(self):
        m = np.asarray(self.matrix, dtype=float)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ValueError(f"reference tensor must be square, got shape {m.shape}")
        if not np.allclose(m, m.T, rtol=0, atol=1e-12 * max(1.0, np.abs(m).max())):
            raise ValueError("reference tensor must be symmetric")
        eigs = np.linalg.eigvalsh(m)
        if eigs[0] <= 0:
            raise ValueError(f"reference tensor must be positive definite, eigs={eigs}")
        object.__setattr__(self, "matrix", m)
        if self.scalar_mode is not None:
            lam = float(self.scalar_mode)
            if lam <= 0 or not np.allclose(m, lam * np.eye(m.shape[0])):
                raise ValueError("scalar_mode inconsistent with matrix")
            object.__setattr__(self, "scalar_mode", lam)

    @classmethod
    def scalar(cls, lam, dim):
        lam = float(lam)
        return cls(lam * np.eye(dim), scalar_mode=lam)

    @property
    def dim(self):
        return self.matrix.shape[0]

    @property
    def c_bound(self):
        return float(np.linalg.eigvalsh(self.matrix)[0])

    @property
    def C_bound(self):
        return float(np.linalg.eigvalsh(self.matrix)[-1])

    @property
    def contrast(self):
        return self.C_bound / self.c_bound
