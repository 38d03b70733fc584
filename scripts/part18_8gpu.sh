#!/bin/bash
# BASELINE config 5 on one 8-GPU node: n = 2^18 int8 NSUM8, level-5 sub-gasket partition,
# tiled per-rank storage, one process per GPU.  Prints one bench line per variant:
#   NCCL all_gather halo (the collective baseline), peer-memory puts, and the exchange fused
#   into the step kernel; 1 and 6 CA steps per exchange.
#   usage: bash scripts/part18_8gpu.sh [NGPUS] [OUT]
N=${1:-8}; OUT=${2:-gpurun_out/part18_${N}gpu.jsonl}
mkdir -p "$(dirname "$OUT")"; : > "$OUT"
for T in 1 6; do
  for HALO in collective peer peer-fused; do
    python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
      --master-port $((29500 + T)) bench.py --gpus "$N" --steps 50 --warmup 5 --workload part18 \
      --halo $HALO --temporal $T --storage tiled | grep '^{' >> "$OUT"
  done
done
python bench.py --workload part18 --steps 50 --warmup 5 --temporal 1 --storage tiled --project 2,4,8 | grep '^{' >> "$OUT"
python bench.py --workload part18 --steps 50 --warmup 5 --temporal 6 --storage tiled --project 2,4,8 | grep '^{' >> "$OUT"
echo "wrote $OUT"
