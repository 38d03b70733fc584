# usage (on the GPU box): LIBS="A B" TS="2 4 6" bash scripts/tb_ab.sh TAG -- fused CA launch times per A/B build (ab/libX.so)
TAG=$1; mkdir -p gpurun_out/$TAG; O=gpurun_out/$TAG/ab.txt
for rep in 1 2; do for L in ${LIBS:-C F2}; do for T in ${TS:-2 4}; do
  echo "== lib$L T=$T" >> $O
  CAPAIR_REPS=1 CAPAIR_STEPS=$T CAPAIR_PROBES=$PROBES GASKET_B200_LIB=ab/lib$L.so timeout 300 python scripts/variants.py capair >> $O 2>&1
done; done; done
