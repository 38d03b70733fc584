# usage (on the GPU box): LIBS="C F" WL=ca17 KREGEX=stencil_tb bash scripts/occ_ab.sh TAG
# per A/B library build (ab/libX.so): occupancy line and one `ncu --set full` capture
TAG=$1
mkdir -p gpurun_out/$TAG
for L in ${LIBS:-C F}; do
  echo "== lib$L" >> gpurun_out/$TAG/occ.txt
  GASKET_DEBUG_OCC=1 GASKET_B200_LIB=ab/lib$L.so timeout 300 python scripts/one_launch.py ${WL:-ca17} 0 2 >> gpurun_out/$TAG/occ.txt 2>&1
  GASKET_B200_LIB=ab/lib$L.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-stencil_tb} -s 1 -c 1 \
    -o gpurun_out/$TAG/lib$L python scripts/one_launch.py ${WL:-ca17} 0 2 >> gpurun_out/$TAG/occ.txt 2>&1
done
