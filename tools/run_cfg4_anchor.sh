set -x
free -g
python tests/golden/make_cfg4_anchor.py labels /tmp/cfg4_labels.npy > gpurun_out/anchor.log 2>&1 || exit 1
(ulimit -v 170000000; python tests/golden/make_cfg4_anchor.py solve /tmp/cfg4_labels.npy gpurun_out/cfg4_729_anchor.npz >> gpurun_out/anchor.log 2>&1) || exit 2
cp gpurun_out/cfg4_729_anchor.npz tests/golden/
PARITY_LOG=gpurun_out/parity_anchor.jsonl python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k anchor > gpurun_out/anchor_test.log 2>&1
tail -3 gpurun_out/anchor_test.log
