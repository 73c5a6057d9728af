#!/bin/bash
# Round 2: ncu --set full of the c3 light kernels at p = 8 (L2-resident v side) for the limiter.
T=${1:-r2aq}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tc_light" -s 2 -c 2 \
    -o gpurun_out/prof_c3p8_$T -f \
    python bench.py --steps 1 --warmup 1 --config c3 --p 8 --light-held 15 --no-e2e --no-cpu > gpurun_out/ncu_c3p8_$T.log 2>&1
tail -2 gpurun_out/ncu_c3p8_$T.log
