#!/bin/bash
# Round 2: c5 grid sweep with MID orientation (p = 12/20/24/32), and the c4 light-kernel ncu capture.
T=${1:-r2aj}
mkdir -p gpurun_out
bash tools/gpu_sweep.sh $T "c5:12 c5:20 c5:24 c5:32"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tc_light" -s 1 -c 1 -o gpurun_out/prof_c4$T -f python bench.py --steps 1 --warmup 1 --config c4 --no-e2e --no-cpu > gpurun_out/ncu_full_c4$T.log 2>&1
tail -n 1 gpurun_out/ncu_full_c4$T.log
