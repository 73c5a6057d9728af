#!/bin/bash
# Round 2: ncu --set full (with source) of the light kernel on c3 (p = 16) and the heavy kernel on c3 at p = 1.
T=${1:-r2aa}
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_tc_light" -s 1 -c 1 -o gpurun_out/prof_c3light$T -f python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_c3light$T.log 2>&1
tail -n 1 gpurun_out/ncu_c3light$T.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_tc_rows" -s 1 -c 1 -o gpurun_out/prof_c3p1rows$T -f python bench.py --config c3 --p 1 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_c3p1rows$T.log 2>&1
tail -n 1 gpurun_out/ncu_c3p1rows$T.log
