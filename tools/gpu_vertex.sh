#!/bin/bash
# per-vertex path: GPU tests + bench lines (usage: bash tools/gpu_vertex.sh <tag>)
T=${1:-v}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_vertex.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_vtx_$T.log 2>&1; tail -15 gpurun_out/pytest_vtx_$T.log
for c in c2 c3 c5; do
  timeout 900 python bench.py --config $c --path vertex --steps 3 --warmup 3 > gpurun_out/bench_vtx_$c$T.json 2> gpurun_out/bench_vtx_$c$T.err
  cut -c1-300 gpurun_out/bench_vtx_$c$T.json; tail -2 gpurun_out/bench_vtx_$c$T.err
done
