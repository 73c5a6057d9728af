#!/bin/bash
# Round 2: medium rows only against short list blocks (R29); c3 p sweep 4..8, c2, c5.
T=${1:-r2ao}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "light_held" > gpurun_out/${T}_tests.log 2>&1; tail -1 gpurun_out/${T}_tests.log
BARGS="--light-held 15" bash tools/gpu_sweep.sh ${T}l15 "c2:8 c3:4 c3:5 c3:6 c3:7 c3:8 c5:16"
BARGS="--light-held 8" bash tools/gpu_sweep.sh ${T}l8 "c2:8 c3:6"
