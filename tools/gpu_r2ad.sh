#!/bin/bash
# Round 2: one list load per lane per round + carried segment index -- parity, timings.
T=${1:-r2ad}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_orient.py tests/test_gpu_vertex.py -q -x -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1; tail -n 2 gpurun_out/pytest_$T.log
bash tools/gpu_sweep.sh $T "c2:8 c5:16 c3:16 c4:1"
