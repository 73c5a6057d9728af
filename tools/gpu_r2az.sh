#!/bin/bash
# Round 2 final evidence (re-run of r2ay without the test suite; r2ay's outputs exceeded gpurun's 64 MiB
# return limit): bench lines + launch lists + ncu --set full per config, summarised ON THE BOX by
# tools/make_profile.py into gpurun_out/profiles_out/ (the .ncu-rep files are not brought back).
T=${1:-r2az}
mkdir -p gpurun_out/profiles_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$T.txt
for c in c5 c3 c2 c4; do bash tools/gpu_bench_profile.sh $c ${c}$T > /dev/null 2>&1; cut -c1-200 gpurun_out/bench_${c}$T.json; done
timeout 900 ncu --set full --clock-control none -k regex:"k_tc_light" -s 2 -c 2 \
    -o gpurun_out/prof_c3L$T -f python bench.py --steps 1 --warmup 1 --config c3 --no-e2e --no-cpu > gpurun_out/ncu_c3L$T.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_tc_light" -s 1 -c 1 \
    -o gpurun_out/prof_c5L$T -f python bench.py --steps 1 --warmup 1 --config c5 --no-e2e --no-cpu > gpurun_out/ncu_c5L$T.log 2>&1
for c in c5 c3 c2 c4; do python tools/make_profile.py ${c}$T $c 02 > /dev/null 2>&1; done
python tools/make_profile.py c3L$T c3 02 > /dev/null 2>&1
python tools/make_profile.py c5L$T c5 02 > /dev/null 2>&1
cp profiles/ncu_summary.json profiles/r02_*$T.json gpurun_out/profiles_out/
rm -f gpurun_out/*.ncu-rep
for c in c2 c5; do
  timeout 900 python bench.py --config $c --path vertex --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_vtx_${c}_$T.json 2> gpurun_out/bench_vtx_${c}_$T.err
  timeout 900 python bench.py --config $c --path cc --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_cc_${c}_$T.json 2> gpurun_out/bench_cc_${c}_$T.err
done
timeout 900 python bench.py --config c5 --budget-gb 16 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c5b16_$T.json 2> gpurun_out/bench_c5b16_$T.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_$T.json 2> gpurun_out/ref_$T.err
du -sh gpurun_out
