#!/bin/bash
# Round 2: medium rows only with scanned lists (R29); c2/c3/c5 with light_held 15; ncu of the c3 p=4 light kernels.
T=${1:-r2an}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "light_held or er_grid or streaming or rmat" > gpurun_out/${T}_tests.log 2>&1; tail -1 gpurun_out/${T}_tests.log
BARGS="--light-held 15" bash tools/gpu_sweep.sh ${T}l15 "c2:8 c3:4 c5:16"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tc_light" -s 2 -c 2 \
    -o gpurun_out/prof_c3p4_$T -f \
    python bench.py --steps 1 --warmup 1 --config c3 --p 4 --light-held 15 --no-e2e --no-cpu > gpurun_out/ncu_c3p4_$T.log 2>&1
tail -2 gpurun_out/ncu_c3p4_$T.log
