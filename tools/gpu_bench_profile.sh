#!/bin/bash
# One GPU call: bench line, launch list, and one full ncu capture of the top kernel.
# usage: bash tools/gpu_bench_profile.sh [config] [tag]
CFG=${1:-c2}
TAG=${2:-$CFG}
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --config "$CFG" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --config "$CFG" --no-e2e --no-cpu > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tc_(rows|light)" -s 2 -c 2 \
    -o gpurun_out/prof_$TAG -f \
    python bench.py --steps 1 --warmup 1 --config "$CFG" --no-e2e --no-cpu > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/ncu_full_$TAG.log
