#!/bin/bash
# Round 2: sector-aligned row slots for short-list blocks (R30): parity, then A/B vs noell on c3/c4/c2.
T=${1:-r2ax}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "light_held or er_grid or closed_forms or rmat or c3 or degenerate or logical or task_times" > gpurun_out/${T}_tests.log 2>&1; tail -1 gpurun_out/${T}_tests.log; grep -m3 "Error\|assert" gpurun_out/${T}_tests.log
bash tools/gpu_ab.sh "noell" "c3:4 c3:6 c3:8 c4:1 c2:8"
