#!/bin/bash
# key counters of one launch of a kernel (regex) in the cfg2 bench: tools/ncu_metrics.sh regex [skip]
k=$1; s=${2:-5}
ncu --clock-control none -k "regex:$k" -s "$s" -c 1 --csv --metrics \
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum \
python bench.py --no-cpu --steps 1 --warmup 3 2>/dev/null | grep -v "^==" | python -c "
import sys, csv
rows = list(csv.reader(sys.stdin))
for r in rows[1:]:
    if len(r) > 14: print(r[4][:40], r[12], r[14], r[13])
"
