#!/bin/bash
# Run the reference's own test suite (pkg/tests, 232 tests) with its hot path
# routed through the GPU (paper_1311_0089_b200.refshim).  Stage the reference
# in the build container first (git-ignored; travels to the GPU box with gpurun):
#   bash tools/run_reference_suite.sh stage
# then on the GPU box:
#   bash tools/run_reference_suite.sh run [pytest args]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
if [ "$1" = "stage" ]; then
  rm -rf "$ROOT/baseline/ref_suite"
  mkdir -p "$ROOT/baseline/ref_suite/src"
  cp -r /root/reference/pkg/src/fftcell "$ROOT/baseline/ref_suite/src/"
  cp -r /root/reference/pkg/tests "$ROOT/baseline/ref_suite/tests"
  find "$ROOT/baseline/ref_suite" -name __pycache__ -prune -exec rm -rf {} +
  echo "staged $(ls "$ROOT/baseline/ref_suite/tests" | wc -l) files"
  exit 0
fi
shift || true
cd "$ROOT/baseline/ref_suite"
PYTHONPATH="$ROOT/baseline/ref_suite/src:$ROOT" python -m pytest -p paper_1311_0089_b200.refshim_pytest tests \
  -p no:cacheprovider -q -rfE "$@"
