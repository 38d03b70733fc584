# usage (on the GPU box): bash scripts/tb_sweep.sh TAG  -- fused-CA staging position / delay sweep
TAG=$1; mkdir -p gpurun_out/$TAG; O=gpurun_out/$TAG/sweep.txt
for T in 2 4; do
  for A in 0 1 2 3; do
    [ $A -ge $T ] && [ $A -ne 0 ] && continue
    for Z in 0 150 300 500; do
      echo "== T=$T stage_at=$A sleep=$Z" >> $O
      CAPAIR_STEPS=$T GASKET_TB_STAGE_AT=$A GASKET_TB_SLEEP=$Z timeout 300 python scripts/variants.py capair 2>&1 | head -2 >> $O
    done
  done
done
