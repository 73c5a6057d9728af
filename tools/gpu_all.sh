#!/bin/bash
# Full round measurement: GPU tests, smoke, c2 bench + launch list + ncu, c3/c4/c5 bench lines.
# usage: bash tools/gpu_all.sh <tag>
T=${1:-v}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$T.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; tail -3 gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/gpu_bench_profile.sh c2 c2$T
for c in c3 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c$T.json 2> gpurun_out/bench_$c$T.err
  cut -c1-300 gpurun_out/bench_$c$T.json; tail -1 gpurun_out/bench_$c$T.err
done
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --cpu-seconds 20 > gpurun_out/bench_c5$T.json 2> gpurun_out/bench_c5$T.err
cut -c1-300 gpurun_out/bench_c5$T.json; tail -2 gpurun_out/bench_c5$T.err
