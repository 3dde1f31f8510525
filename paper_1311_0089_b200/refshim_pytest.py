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


def pytest_terminal_summary(terminalreporter):
    calls = ", ".join(f"{k} {v}" for k, v in refshim.CALLS.items())
    terminalreporter.write_line(f"B200 shim: hot-path calls routed to the GPU: {calls}")
