# A/B of the deferred x update (FC_DEFER_X) on cfg2 and cfg3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
bash tools/tune.sh "FC_DEFER_X=0" "FC_DEFER_X=1" "FC_DEFER_X=0" "FC_DEFER_X=1" 2>&1 | tee gpurun_out/ab_defer.log
for v in 0 1; do FC_DEFER_X=$v timeout 300 python bench.py --no-cpu --config cfg3 --steps 3 --warmup 3 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg3 defer=$v', d['value'], d['iteration_roofline'], {n: round(v['avg_ms'],4) for n,v in d['kernels'].items()})"; done 2>&1 | tee -a gpurun_out/ab_defer.log
