#!/bin/bash
# Round 2: ncu --set full of the thread-per-row kernels alone: c3 (light <8> + medium <15> of one count) and c5 (light).
T=${1:-r2av}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tc_light" -s 2 -c 2 \
    -o gpurun_out/prof_c3L$T -f python bench.py --steps 1 --warmup 1 --config c3 --no-e2e --no-cpu > gpurun_out/ncu_c3L$T.log 2>&1
tail -1 gpurun_out/ncu_c3L$T.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tc_light" -s 1 -c 1 \
    -o gpurun_out/prof_c5L$T -f python bench.py --steps 1 --warmup 1 --config c5 --no-e2e --no-cpu > gpurun_out/ncu_c5L$T.log 2>&1
tail -1 gpurun_out/ncu_c5L$T.log
