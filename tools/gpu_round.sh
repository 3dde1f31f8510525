# tests, bench line, reference arm, ncu launch list and full capture of the CG kernels
# usage: bash tools/gpu_round.sh TAG
t=${1:-rxx}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | tee gpurun_out/${t}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${t}_bench.log 2>&1; grep '^{' gpurun_out/${t}_bench.log > gpurun_out/${t}_bench.json; tail -c 600 gpurun_out/${t}_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | grep '^{' > gpurun_out/${t}_reference_arm.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${t}_launches.csv \
  python bench.py --no-cpu --steps 2 --warmup 3 > gpurun_out/${t}_ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_row_fwd|k_outer|k_row_inv|k_cg_update" -s 40 -c 4 \
  -o gpurun_out/${t}_full -f python bench.py --no-cpu --steps 1 --warmup 3 > gpurun_out/${t}_ncu_full.log 2>&1; echo "full rc=$?"
timeout 600 python bench.py --no-cpu --config cfg3 --steps 3 --warmup 3 2>&1 | grep '^{' > gpurun_out/${t}_bench_cfg3.json
timeout 900 python bench.py --no-cpu --config cfg4 --steps 1 --warmup 1 2>&1 | grep '^{' > gpurun_out/${t}_bench_cfg4.json
timeout 600 python tools/fp_bench.py 243 2>&1 | tail -3 > gpurun_out/${t}_fp_cfg3.log
