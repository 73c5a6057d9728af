#!/bin/bash
# Round 2: c5 grid sweep below p = 16 (p = 6..14), MID orientation.
T=${1:-r2ak}
mkdir -p gpurun_out
bash tools/gpu_sweep.sh $T "c5:6 c5:8 c5:10 c5:12 c5:14"
