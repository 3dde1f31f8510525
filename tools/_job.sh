set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02q_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02q_pytest_gpu.log
tail -4 gpurun_out/r02q_pytest_gpu.log
timeout 900 python tools/ab_plan.py cfg4 0 "" > gpurun_out/r02q_ab_cfg4.txt 2>&1; cat gpurun_out/r02q_ab_cfg4.txt
timeout 900 python tools/ab_plan.py cfg2 0 "" > gpurun_out/r02q_ab_cfg2.txt 2>&1; cat gpurun_out/r02q_ab_cfg2.txt
