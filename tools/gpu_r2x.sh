#!/bin/bash
# Round 2: c3 p sweep (per-kernel split, item counts) to pick the block grid for uniform sparse graphs.
T=${1:-r2x}
mkdir -p gpurun_out
bash tools/gpu_sweep.sh $T "c3:1 c3:2 c3:4 c3:8 c3:16 c2:4 c2:16"
