#!/bin/bash
# tests + c2 bench/profile + c5 bench + c5s ncu capture.  usage: bash tools/gpu_round.sh <tag>
T=${1:-v}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
bash tools/gpu_bench_profile.sh c2 c2$T
timeout 600 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c5$T.json 2> gpurun_out/bench_c5$T.err
cut -c1-400 gpurun_out/bench_c5$T.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_rows -s 1 -c 1 -o gpurun_out/prof_c5s$T -f \
    python bench.py --config c5s --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_c5s$T.log 2>&1
tail -2 gpurun_out/ncu_full_c5s$T.log
