#!/bin/bash
# Round 2: light kernel 16-byte chunk scans (PGABB_LIGHT_VEC, default) vs held-id chunks (avec) vs scalar (novec).
T=${1:-r2ar}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "light_held or er_grid or closed_forms or rmat or streaming or degenerate" > gpurun_out/${T}_tests.log 2>&1; tail -1 gpurun_out/${T}_tests.log
bash tools/gpu_ab.sh "avec novec" "c3:4 c3:8 c4:1 c2:8"
