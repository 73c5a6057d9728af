#!/bin/bash
# Round 2: per-path cycle shares of the counting vs the per-vertex (VM = 3) heavy kernel.
T=${1:-r2ab}
mkdir -p gpurun_out
timeout 900 python tools/prof_paths.py run c2 c2:vertex c5s c5s:vertex > gpurun_out/paths_$T.json 2> gpurun_out/paths_$T.err
cat gpurun_out/paths_$T.json; tail -2 gpurun_out/paths_$T.err
