#!/bin/bash
# Round 2: light kernel evict-first streaming loads (cs) and 8 CTAs/SM (m8) A/B on c3 p = 4..8, c4, c2.
T=${1:-r2as}
mkdir -p gpurun_out
bash tools/gpu_ab.sh "cs m8" "c3:4 c3:6 c3:8 c4:1 c2:8"
