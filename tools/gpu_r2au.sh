#!/bin/bash
# Round 2: medium-kernel occupancy A/B (4 / 5 / 6 CTAs/SM) on c3; per-vertex kernel at 5 CTAs/SM (vtx5);
# per-path cycle shares of the per-vertex heavy kernel (prof build).
T=${1:-r2au}
mkdir -p gpurun_out
bash tools/gpu_ab.sh "med4 med6" "c3:4"
BARGS="--path vertex" bash tools/gpu_sweep.sh ${T}vd "c2:8 c5:16"
BARGS="--path vertex" PGABB_LIB_VARIANT=vtx5 bash tools/gpu_sweep.sh ${T}v5 "c2:8 c5:16"
timeout 900 python tools/prof_paths.py run c2:vertex c5:vertex c2 > gpurun_out/paths_$T.json 2> gpurun_out/paths_$T.err; cut -c1-700 gpurun_out/paths_$T.json
