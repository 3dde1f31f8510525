set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02o_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02o_pytest_gpu.log
tail -4 gpurun_out/r02o_pytest_gpu.log
timeout 600 python tools/ab_plan.py cfg3 0 "" > gpurun_out/r02o_ab_cfg3.txt 2>&1
cat gpurun_out/r02o_ab_cfg3.txt
python -c "import __graft_entry__ as g; g.smoke()"
