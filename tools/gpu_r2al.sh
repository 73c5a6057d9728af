#!/bin/bash
# Round 2: c3 grid sweep with the light kernel at 8 vs 15 held ids.
T=${1:-r2al}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
bash tools/gpu_sweep.sh ${T}d "c3:1 c3:2 c3:4 c3:8 c3:16"
PGABB_LIB_VARIANT=la15 bash tools/gpu_sweep.sh ${T}la15 "c3:2 c3:4 c3:8 c3:16 c4:1 c2:8"
