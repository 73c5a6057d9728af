#!/bin/bash
# one tuning iteration: GPU parity tests, c2/c5 bench lines, per-path cycle shares
T=${1:-v}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
python bench.py --config c2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c2$T.json 2> gpurun_out/bench_c2$T.err
cut -c1-250 gpurun_out/bench_c2$T.json; tail -2 gpurun_out/bench_c2$T.err
timeout 600 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c5$T.json 2> gpurun_out/bench_c5$T.err
cut -c1-250 gpurun_out/bench_c5$T.json; tail -2 gpurun_out/bench_c5$T.err
timeout 900 python tools/prof_paths.py run ${PATHS_CFGS:-c2 c5} > gpurun_out/paths_$T.jsonl 2> gpurun_out/paths_$T.err
cat gpurun_out/paths_$T.jsonl; tail -2 gpurun_out/paths_$T.err
