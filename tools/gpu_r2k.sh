#!/bin/bash
# Round 2: ncu --set full of the light kernel on c3 (LOW, p=16) and c4 (p=1), with source.
T=${1:-r2k}
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_tc_light" -s 1 -c 1 -o gpurun_out/prof_c3light$T -f python bench.py --config c3 --orient low --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_c3light$T.log 2>&1
tail -n 1 gpurun_out/ncu_c3light$T.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_tc_light" -s 1 -c 1 -o gpurun_out/prof_c4light$T -f python bench.py --config c4 --p 1 --orient low --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_c4light$T.log 2>&1
tail -n 1 gpurun_out/ncu_c4light$T.log
