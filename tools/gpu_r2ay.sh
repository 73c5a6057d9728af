#!/bin/bash
# Round 2 final measurement after R30 (sector-aligned slots): full GPU suite, smoke, bench lines + launch
# lists + ncu --set full of both S10 kernels on c5/c2/c3/c4, thread-kernel-only captures for c3/c5,
# per-vertex and cc lines, streamed c5, reference arm.
T=${1:-r2ay}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$T.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; tail -n 2 gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
for c in c5 c3 c2 c4; do bash tools/gpu_bench_profile.sh $c ${c}$T > /dev/null 2>&1; cut -c1-220 gpurun_out/bench_${c}$T.json; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tc_light" -s 2 -c 2 \
    -o gpurun_out/prof_c3L$T -f python bench.py --steps 1 --warmup 1 --config c3 --no-e2e --no-cpu > gpurun_out/ncu_c3L$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tc_light" -s 1 -c 1 \
    -o gpurun_out/prof_c5L$T -f python bench.py --steps 1 --warmup 1 --config c5 --no-e2e --no-cpu > gpurun_out/ncu_c5L$T.log 2>&1
for c in c2 c5; do
  timeout 900 python bench.py --config $c --path vertex --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_vtx_${c}_$T.json 2> gpurun_out/bench_vtx_${c}_$T.err
  timeout 900 python bench.py --config $c --path cc --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_cc_${c}_$T.json 2> gpurun_out/bench_cc_${c}_$T.err
  cut -c1-160 gpurun_out/bench_vtx_${c}_$T.json gpurun_out/bench_cc_${c}_$T.json
done
timeout 900 python bench.py --config c5 --budget-gb 16 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c5b16_$T.json 2> gpurun_out/bench_c5b16_$T.err; cut -c1-160 gpurun_out/bench_c5b16_$T.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_$T.json 2> gpurun_out/ref_$T.err; cut -c1-200 gpurun_out/ref_$T.json
