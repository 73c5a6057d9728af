#!/bin/bash
# Round 2: light_held auto (R29): full GPU suite, then c2/c3/c4/c5 with the auto rule.
T=${1:-r2ap}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; tail -n 2 gpurun_out/pytest_gpu_$T.log
bash tools/gpu_sweep.sh ${T} "c2:8 c3:4 c4:1 c5:16"
