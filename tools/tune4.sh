#!/bin/bash
# usage: tools/tune4.sh "ENV=a" ...   (one-step cfg4 bench per setting)
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 600 python bench.py --no-cpu --config cfg4 --steps 1 --warmup 1 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.4e'%d['value'], d['iterations'], round(d['iteration_roofline']['ms'],3), {k: round(v['avg_ms'],3) for k,v in d['kernels'].items()})"
done
