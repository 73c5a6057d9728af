#!/bin/bash
# Round 2: heavy-kernel knobs re-tuned after the 1-load-per-round list loop (c2, c5s, c5).
T=${1:-r2af}
mkdir -p gpurun_out
for v in "" nofilt and1 and4 chunk8 minb6; do
  echo "== variant ${v:-default}"
  PGABB_LIB_VARIANT=$v bash tools/gpu_sweep.sh $T$v "c2:8 c5s:16 c5:16"
done
