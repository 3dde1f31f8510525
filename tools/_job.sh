set -x
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r02p_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02p_pytest.log
tail -8 gpurun_out/r02p_pytest.log
timeout 900 python tools/ab_plan.py cfg4 0 "" "outer_par=1" "outer_par=1,outer_threads=162" > gpurun_out/r02p_ab_outer_par_cfg4.txt 2>&1
cat gpurun_out/r02p_ab_outer_par_cfg4.txt
timeout 600 python tools/ab_plan.py cfg3 0 "" "outer_par=1" "outer_par=1,outer_threads=108" "outer_par=1,outer_threads=243" > gpurun_out/r02p_ab_outer_par_cfg3.txt 2>&1
cat gpurun_out/r02p_ab_outer_par_cfg3.txt
timeout 600 python tools/ab_plan.py cfg2 0 "" "outer_par=1" > gpurun_out/r02p_ab_outer_par_cfg2.txt 2>&1
cat gpurun_out/r02p_ab_outer_par_cfg2.txt
