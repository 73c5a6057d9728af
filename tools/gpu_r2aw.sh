#!/bin/bash
# Round 2: medium rows that binary-search long lists (medlong) vs scanned-only, c3 p = 4 / 8.
T=${1:-r2aw}
mkdir -p gpurun_out
bash tools/gpu_ab.sh "medlong" "c3:4 c3:8"
