#!/bin/bash
# Round 2: heavy-kernel A/B -- dense-copy threshold 1/64, 1/128 and 1/4/2 list loads in flight.
T=${1:-r2ac}
mkdir -p gpurun_out
for v in "" d64 d128 u4 u1; do
  echo "== variant ${v:-default}"
  PGABB_LIB_VARIANT=$v bash tools/gpu_sweep.sh $T$v "c2:8 c5:16 c3:16"
done
