set -x
timeout 1200 python -m pytest tests/test_gpu_fat.py -m gpu -x -q > gpurun_out/r02j_pytest_fat.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02j_pytest_fat.log
tail -30 gpurun_out/r02j_pytest_fat.log
timeout 900 python tools/ab_plan.py cfg4 0 "" "outer_direct=1" "outer_direct=1,outer_threads=162" > gpurun_out/r02j_ab_outer_direct_cfg4.txt 2>&1
cat gpurun_out/r02j_ab_outer_direct_cfg4.txt
timeout 600 python tools/ab_plan.py cfg3 0 "" "outer_direct=1" "outer_direct=1,outer_threads=108" "outer_direct=1,outer_threads=243"  > gpurun_out/r02j_ab_outer_direct_cfg3.txt 2>&1
cat gpurun_out/r02j_ab_outer_direct_cfg3.txt
