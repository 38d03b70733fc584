#!/bin/bash
# usage (on the GPU box): bash scripts/ncu_dram.sh OUT WORKLOAD KERNEL_REGEX FLAGS...
#   per-launch DRAM bytes and duration (ncu, cold cache) of scripts/one_launch.py's second
#   launch for each flag set: the traffic check of a variant (not a timing)
OUT=$1; WL=$2; K=$3; shift 3
for F in "$@"; do
  echo "== $WL flags=$F"
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_write.sum \
    --clock-control none -k regex:$K -s 1 -c 1 --csv python scripts/one_launch.py $WL $F 2 2>/dev/null | grep -E '"(dram|gpu__|lts)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done > $OUT 2>&1
