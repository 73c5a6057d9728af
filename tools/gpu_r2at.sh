#!/bin/bash
# Round 2 measurement of HEAD (after R29 medium rows): full GPU suite, smoke, sanitizers, bench lines + launch lists + ncu --set full
# of both S10 kernels on c5 (default), c2, c3, c4; per-vertex and cc lines; streamed c5; reference arm.
T=${1:-r2at}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$T.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; tail -n 2 gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/memcheck_$T.log 2>&1; tail -n 2 gpurun_out/memcheck_$T.log
timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_run.py > gpurun_out/racecheck_$T.log 2>&1; tail -n 2 gpurun_out/racecheck_$T.log
for c in c5 c2 c3 c4; do bash tools/gpu_bench_profile.sh $c ${c}$T > /dev/null 2>&1; cut -c1-220 gpurun_out/bench_${c}$T.json; done
for c in c2 c5; do
  timeout 900 python bench.py --config $c --path vertex --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_vtx_${c}_$T.json 2> gpurun_out/bench_vtx_${c}_$T.err
  timeout 900 python bench.py --config $c --path cc --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_cc_${c}_$T.json 2> gpurun_out/bench_cc_${c}_$T.err
  cut -c1-160 gpurun_out/bench_vtx_${c}_$T.json gpurun_out/bench_cc_${c}_$T.json
done
timeout 900 python bench.py --config c5 --budget-gb 16 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c5b16_$T.json 2> gpurun_out/bench_c5b16_$T.err; cut -c1-160 gpurun_out/bench_c5b16_$T.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_$T.json 2> gpurun_out/ref_$T.err; cut -c1-200 gpurun_out/ref_$T.json
