set -x
python bench.py --steps 2 --warmup 1 --no-cpu --no-others > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02c.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-others > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_(row|mid|outer|cg)" -s 12 -c 6 -o gpurun_out/r02c_cfg4_full python tools/ncu_solve.py cfg4 4 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out/
