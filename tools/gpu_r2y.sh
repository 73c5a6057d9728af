#!/bin/bash
# Round 2: light-row width variants on c3 (p = 1/2/4) + regressions, and per-path cycle shares
# of the count vs the per-vertex (VM=3) heavy kernel.
T=${1:-r2y}
mkdir -p gpurun_out
for v in "" la15w256 la15w1k la8w512; do
  echo "== variant ${v:-default}"
  PGABB_LIB_VARIANT=$v bash tools/gpu_sweep.sh $T$v "c3:1 c3:2 c3:4 c4:1 c2:8 c5:16"
done
timeout 900 python tools/prof_paths.py run c2 c2:vertex c5s c5s:vertex > gpurun_out/paths_$T.json 2> gpurun_out/paths_$T.err
cat gpurun_out/paths_$T.json; tail -2 gpurun_out/paths_$T.err
