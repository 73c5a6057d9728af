#!/bin/bash
# Round 2: ncu --set full of the c5 k_tc_rows (auto orientation) with source lines.
T=${1:-r2i}
mkdir -p gpurun_out
timeout 2400 ncu --set full --import-source on --clock-control none -k regex:"k_tc_rows" -c 1 -o gpurun_out/prof_c5$T -f python bench.py --config c5 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full_c5$T.log 2>&1
tail -n 2 gpurun_out/ncu_full_c5$T.log
