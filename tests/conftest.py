"""Shared fixtures.  ``gpu``-marked tests need a B200 (run with ``-m gpu``);
everything else runs on CPU.  Helpers mirror the reference's
``pkg/tests/conftest.py`` so the parity tests read like the reference's own."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    path = GOLDEN / f"{name}.npz"
    if not path.exists():
        pytest.skip(f"golden fixture {name}.npz not generated")
    return np.load(path, allow_pickle=False)


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def random_spd_packed(shape, rng, shift=0.5):
    """B B^T + shift I per point, packed (reference conftest.py:28-34)."""
    d = len(shape)
    B = rng.standard_normal((d, d) + tuple(shape))
    mats = np.einsum("ab...,cb...->ac...", B, B) + shift * np.eye(d).reshape((d, d) + (1,) * d)
    pairs = [(a, a) for a in range(d)] + [(a, b) for a in range(d) for b in range(a + 1, d)]
    return np.stack([mats[a, b] for a, b in pairs])


def random_gradient_field(shape, Y, rng):
    """Curl-free zero-mean field (reference conftest.py:37-49)."""
    from oracle.fftcell_oracle import frequency_grid

    d = len(shape)
    p = rng.standard_normal(shape)
    vhat = 1j * np.pi * frequency_grid(shape, Y) * np.fft.fftn(p)[np.newaxis]
    vhat[(slice(None),) + (0,) * d] = 0.0
    return np.fft.ifftn(vhat, axes=tuple(range(1, d + 1))).real


def mean_residual(values):
    d = values.shape[0]
    return float(np.max(np.abs(values.reshape(d, -1).mean(axis=1))))


def curl_residual(values, Y):
    """Largest Fourier component orthogonal to xi(k) (reference conftest.py:71-82)."""
    from oracle.fftcell_oracle import frequency_grid

    d = values.shape[0]
    shape = values.shape[1:]
    axes = tuple(range(1, d + 1))
    vhat = np.fft.fftn(values, axes=axes) / np.prod(shape)
    xi = frequency_grid(shape, Y)
    norm2 = np.einsum("a...,a...->...", xi, xi)
    norm2[(0,) * d] = 1.0
    dots = np.einsum("a...,a...->...", xi, vhat)
    ortho = vhat - xi * (dots / norm2)[np.newaxis]
    ortho[(slice(None),) + (0,) * d] = 0.0
    return float(np.max(np.abs(ortho)))


def rel_l2(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def log_parity(rec):
    """Append a parity record (margins vs gates) to $PARITY_LOG when set."""
    import json
    import os

    path = os.environ.get("PARITY_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(rec) + "\n")
