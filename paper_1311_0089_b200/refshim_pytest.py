"""pytest plugin: run the reference's own test suite against the B200 path.

    PYTHONPATH=<reference src>:<repo> python -m pytest -p paper_1311_0089_b200.refshim_pytest <reference tests>

Installs ``paper_1311_0089_b200.refshim`` (the hot-path entry points of the
imported ``fftcell`` replaced by GPU wrappers) in ``pytest_configure``, i.e.
before the test modules are collected and bind the names, and reports at the
end how many calls were routed to the GPU.
"""

from __future__ import annotations

from . import refshim


def pytest_configure(config):
    refshim.install()
    # create the CUDA context and load the library's kernels now: the reference's
    # first acceptance test budgets 1 s of wall clock for a solve (test_acceptance.py:43),
    # which should not pay for driver initialisation
    import numpy as np

    from . import _native
    from .grid import GridSpec

    ctx = _native.Context(GridSpec((1.0, 1.0), (9, 9)))
    ctx.project(0, None, np.zeros((1, 2, 9, 9)))  # FC_PROJ_ORTHOGONAL: needs no coefficients
    del ctx


def pytest_terminal_summary(terminalreporter):
    calls = ", ".join(f"{k} {v}" for k, v in refshim.CALLS.items())
    terminalreporter.write_line(f"B200 shim: hot-path calls routed to the GPU: {calls}")
