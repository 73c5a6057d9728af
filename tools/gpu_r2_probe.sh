#!/bin/bash
# Round-2 first probe: box facts, current per-config timings, C5 per-path cycle shares,
# and C5 ncu counters of the two S10 kernels (targeted sections, then --set full).
mkdir -p gpurun_out
T=${1:-p1}
{ nproc; free -g; lscpu | grep -E "Model name|Socket|Thread|Core"; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv; } > gpurun_out/box_$T.txt 2>&1
for c in c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${c}_$T.json 2> gpurun_out/bench_${c}_$T.err
  cut -c1-200 gpurun_out/bench_${c}_$T.json
done
timeout 900 python tools/prof_paths.py run c2 c5s c5 > gpurun_out/paths_$T.json 2> gpurun_out/paths_$T.err
cat gpurun_out/paths_$T.json
timeout 1500 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section LaunchStats --section Occupancy --section SchedulerStats --section ComputeWorkloadAnalysis --clock-control none -k regex:"k_tc_(rows|light)" -c 2 -o gpurun_out/sec_c5$T -f python bench.py --config c5 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_sec_c5$T.log 2>&1
tail -n 3 gpurun_out/ncu_sec_c5$T.log
timeout 2400 ncu --set full --import-source on --clock-control none -k regex:"k_tc_rows" -c 1 -o gpurun_out/prof_c5$T -f python bench.py --config c5 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full_c5$T.log 2>&1
tail -n 3 gpurun_out/ncu_full_c5$T.log
