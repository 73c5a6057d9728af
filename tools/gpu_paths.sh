#!/bin/bash
# per-path cycle shares of k_tc_rows (instrumented build) + bench lines of c3/c4
mkdir -p gpurun_out
T=${1:-v}
timeout 900 python tools/prof_paths.py run c2 c5s c5 c3 c4 > gpurun_out/paths_$T.jsonl 2> gpurun_out/paths_$T.err
tail -3 gpurun_out/paths_$T.err; cat gpurun_out/paths_$T.jsonl
for c in c3 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${c}$T.json 2> gpurun_out/bench_${c}$T.err
  cut -c1-300 gpurun_out/bench_${c}$T.json; tail -2 gpurun_out/bench_${c}$T.err
done
