#!/bin/bash
# usage (on the GPU box): bash scripts/ncu_one.sh TAG WORKLOAD FLAGS KERNEL_REGEX
#   one `ncu --set full` capture of the second launch of scripts/one_launch.py
#   e.g. bash scripts/ncu_one.sh s3 stencil17 2 stencil_v2 ; bash scripts/ncu_one.sh s3 ca17 0 stencil_tb2
TAG=$1; WL=$2; FLAGS=$3; K=$4
mkdir -p gpurun_out/$TAG
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
  -o gpurun_out/$TAG/${WL}_f${FLAGS} python scripts/one_launch.py $WL $FLAGS 2 > gpurun_out/$TAG/ncu_${WL}_f${FLAGS}.log 2>&1
echo ncu_rc=$?
