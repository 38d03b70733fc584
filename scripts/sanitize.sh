#!/bin/bash
# usage (on the GPU box): bash scripts/sanitize.sh OUTDIR
#   compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_cases.py
#   (every product kernel family, small sizes) and the two-process fused peer path
#   bash scripts/sanitize.sh OUTDIR part   -- the two-process peer cases only
OUT=${1:-gpurun_out/sanitize}; mkdir -p $OUT
CS=compute-sanitizer
[ "$2" = "part" ] || for T in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $T --print-limit 20 python scripts/sanitize_cases.py > $OUT/$T.log 2>&1; echo "$T rc=$?" >> $OUT/rc.txt
done
for T in memcheck synccheck; do
  timeout 900 $CS --tool $T --target-processes all --print-limit 20 python scripts/sanitize_cases.py part > $OUT/part_$T.log 2>&1; echo "part_$T rc=$?" >> $OUT/rc.txt
done
