#!/bin/bash
# run a command with an alternative build of the library swapped in (A/B timing)
alt=$1; shift
cp paper_1311_0089_b200/libfftcell_b200.so /tmp/lib_main.so
cp "$alt" paper_1311_0089_b200/libfftcell_b200.so
"$@"
cp /tmp/lib_main.so paper_1311_0089_b200/libfftcell_b200.so
