#!/bin/bash
# Round 2: memory-lean build + 64-bit lift: GPU tests (incl. the 2 x C5 union through a
# budget), default bench, wave trace of c5 through 16 GB.
T=${1:-r2q}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=8 > gpurun_out/pytest_gpu_$T.log 2>&1; tail -n 14 gpurun_out/pytest_gpu_$T.log
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d.get('ms_per_step'), d.get('parity',{}).get('match'), (d.get('e2e') or {}).get('ms_per_step'), d.get('run',{}).get('build_ms'))" $1 "$2" 2>&1 | tail -1; }
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c5_$T.json 2> gpurun_out/bench_c5_$T.err
summ gpurun_out/bench_c5_$T.json "c5"
timeout 900 python tools/wave_trace.py c5 16 > gpurun_out/wave_trace_c5_$T.json 2> gpurun_out/wave_trace_c5_$T.err; tail -n 1 gpurun_out/wave_trace_c5_$T.err
