#!/bin/bash
# A/B the in-tree library against another build on the cfg3 bench: tools/ab3.sh alt.so [rounds]
alt=$1; n=${2:-1}
cp paper_1311_0089_b200/libfftcell_b200.so /tmp/lib_main3.so
show() { grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.4e'%d['value'], round(d['iteration_roofline']['ms'],4), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; }
for i in $(seq "$n"); do
  echo "== main cfg3"; cp /tmp/lib_main3.so paper_1311_0089_b200/libfftcell_b200.so; python bench.py --no-cpu --config cfg3 --steps 3 --warmup 3 2>&1 | show
  echo "== alt cfg3"; cp "$alt" paper_1311_0089_b200/libfftcell_b200.so; python bench.py --no-cpu --config cfg3 --steps 3 --warmup 3 2>&1 | show
done
cp /tmp/lib_main3.so paper_1311_0089_b200/libfftcell_b200.so
