#!/bin/bash
# Round 2: K-slot block cache -- streaming tests + c5 wave traces at several budgets.
T=${1:-r2s}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "stream or budget or union or wave" > gpurun_out/pytest_stream_$T.log 2>&1; tail -n 3 gpurun_out/pytest_stream_$T.log
for b in 16 24 32 48; do
  timeout 900 python tools/wave_trace.py c5 $b > gpurun_out/wave_trace_c5_b${b}_$T.json 2> gpurun_out/wave_trace_c5_b${b}_$T.err; tail -n 1 gpurun_out/wave_trace_c5_b${b}_$T.err
done
