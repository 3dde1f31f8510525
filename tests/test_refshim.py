"""The drop-in shim (paper_1311_0089_b200.refshim) patches the reference's
hot-path entry points and every copy its callers bound at import.  CPU only;
the reference's own 232-test suite runs through it on the GPU with
tools/run_reference_suite.sh (log: profiles/r02_reference_suite_on_gpu.log)."""

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CANDIDATES = [ROOT / "baseline" / "ref_suite" / "src", Path("/root/reference/pkg/src")]
SRC = next((p for p in CANDIDATES if (p / "fftcell").is_dir()), None)


@pytest.mark.skipif(SRC is None, reason="reference package not available")
def test_shim_patches_every_bound_name():
    code = f"""
import sys
sys.path[:0] = [{str(SRC)!r}, {str(ROOT)!r}]
import fftcell.solver as S, fftcell.homogenize as H, fftcell.analysis as A, fftcell.cli as C
from paper_1311_0089_b200 import refshim
refshim.install()
assert S.solve_cg.__module__ == refshim.__name__
for mod, names in ((S, ["solve_cg", "solve_neumann", "solve", "apply_system", "_Projector"]),
                   (H, ["solve"]), (A, ["solve_cg", "solve_neumann", "_Projector"]), (C, ["solve"])):
    for n in names:
        assert getattr(mod, n).__module__ == refshim.__name__, (mod.__name__, n)
print("ok")
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr
