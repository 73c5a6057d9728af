#!/bin/bash
# Round 2: medium thread-per-row items (R29): parity, then c3/c2/c4/c5 with light_held 8 vs 15.
T=${1:-r2am}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "light_held or er_grid or streaming or closed_forms or rmat" > gpurun_out/${T}_tests.log 2>&1; tail -3 gpurun_out/${T}_tests.log
BARGS="--light-held 8" bash tools/gpu_sweep.sh ${T}l8 "c3:4 c3:8 c2:8 c4:1 c5:16"
BARGS="--light-held 15" bash tools/gpu_sweep.sh ${T}l15 "c3:2 c3:4 c3:8 c3:16 c2:8 c4:1 c5:16"
