#!/bin/bash
# usage: tools/tune3.sh "ENV=a" ...   (short cfg3 bench per setting)
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg python bench.py --no-cpu --config cfg3 --steps 3 --warmup 3 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.4e'%d['value'], round(d['iteration_roofline']['ms'],4), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"
done
