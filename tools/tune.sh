#!/bin/bash
# usage: tools/tune.sh "ENV1=a ENV2=b" "ENV1=c" ...   (runs a short cfg2 bench per setting)
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg python bench.py --no-cpu --steps 3 --warmup 3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l)
        k = d['kernels']
        print('value %.3e  iter_ms %.3f  frac %.3f' % (d['value'], d['iteration_roofline']['ms'], d['iteration_roofline']['frac']))
        print('   ', {n: round(v['avg_ms'], 4) for n, v in k.items()})
    else:
        sys.stdout.write(l)
"
done
