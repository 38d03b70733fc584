#!/bin/bash
# Two bench ranks sharing one GPU (gloo plumbing), each under its own timeout with a
# Python traceback dump on expiry: diagnoses a hang of tests/test_bench_multirank.py.
# usage: bash scripts/repro_multirank.sh HALO TEMPORAL STORAGE [SECONDS]
HALO=${1:-collective}; T=${2:-1}; ST=${3:-tiled}; SECS=${4:-120}
PORT=$((20000 + RANDOM % 20000))
mkdir -p gpurun_out
for R in 0 1; do
  GASKET_BENCH_SHARED_GPU=1 OMP_NUM_THREADS=1 RANK=$R LOCAL_RANK=$R WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=$PORT \
    timeout -s ABRT $SECS python -X faulthandler bench.py --gpus 2 --steps 4 --warmup 3 --workload part15 \
    --halo $HALO --temporal $T --storage $ST > gpurun_out/mr_${HALO}_${T}_${ST}_r$R.log 2>&1 &
done
wait
tail -c 4000 gpurun_out/mr_${HALO}_${T}_${ST}_r0.log
echo ----
tail -c 4000 gpurun_out/mr_${HALO}_${T}_${ST}_r1.log
