#!/bin/bash
# A/B the in-tree library against another build on the cfg2 bench, interleaved
# on the same box.  usage: tools/ab.sh alt.so [rounds] [ENV=..]
alt=$1; n=${2:-2}; envs=${3:-}
cp paper_1311_0089_b200/libfftcell_b200.so /tmp/lib_main.so
for i in $(seq "$n"); do
  echo "== main"; cp /tmp/lib_main.so paper_1311_0089_b200/libfftcell_b200.so; bash tools/tune.sh "$envs" | tail -2
  echo "== alt $alt"; cp "$alt" paper_1311_0089_b200/libfftcell_b200.so; bash tools/tune.sh "$envs" | tail -2
done
cp /tmp/lib_main.so paper_1311_0089_b200/libfftcell_b200.so
