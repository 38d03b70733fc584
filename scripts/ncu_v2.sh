mkdir -p gpurun_out/s2g
for F in 2 10 24578; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_v2 -s 1 -c 1 -o gpurun_out/s2g/v2_$F python scripts/one_launch.py stencil17 $F 2 > gpurun_out/s2g/ncu_$F.log 2>&1; echo rc=$?
done
