#!/bin/bash
T=${1:-v}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
python bench.py --config c2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c2$T.json 2> gpurun_out/bench_c2$T.err; cut -c1-300 gpurun_out/bench_c2$T.json
timeout 600 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c5$T.json 2> gpurun_out/bench_c5$T.err; cut -c1-300 gpurun_out/bench_c5$T.json
timeout 300 python tools/task_stats.py c5s > gpurun_out/tasks_c5s.json 2>gpurun_out/tasks_c5s.err
timeout 300 python tools/task_stats.py c5 > gpurun_out/tasks_c5.json 2>gpurun_out/tasks_c5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_rows -s 1 -c 1 -o gpurun_out/prof_c5s$T -f \
    python bench.py --config c5s --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_c5s$T.log 2>&1
tail -1 gpurun_out/ncu_full_c5s$T.log
