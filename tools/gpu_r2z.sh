#!/bin/bash
# Round 2: batched small rows in k_tc_rows -- parity tests, then A/B vs no batching / 4 CTAs / batch la <= 16.
T=${1:-r2z}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_orient.py -q -x -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1; tail -n 2 gpurun_out/pytest_$T.log
for v in "" nobatch minb4 b16; do
  echo "== variant ${v:-default}"
  PGABB_LIB_VARIANT=$v bash tools/gpu_sweep.sh $T$v "c3:1 c3:2 c3:4 c4:1 c2:8 c5:16"
done
