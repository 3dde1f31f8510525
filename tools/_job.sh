set -x
timeout 1200 python -m pytest tests/test_gpu_variants.py -m gpu -x -q > gpurun_out/r02r_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02r_pytest.log
tail -4 gpurun_out/r02r_pytest.log
timeout 900 python tools/ab_plan.py cfg4 0 "" "mid_direct=1" "mid_direct=2" "mid_direct=3" > gpurun_out/r02r_ab_mid_direct_cfg4.txt 2>&1; cat gpurun_out/r02r_ab_mid_direct_cfg4.txt
timeout 900 python tools/ab_plan.py cfg3 0 "" "mid_direct=1" "mid_direct=2" "mid_direct=3" > gpurun_out/r02r_ab_mid_direct_cfg3.txt 2>&1; cat gpurun_out/r02r_ab_mid_direct_cfg3.txt
