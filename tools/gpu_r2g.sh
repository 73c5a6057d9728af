#!/bin/bash
# Round 2: cut rules 2/3 (parity + c5 sweep) and the per-path cycle shares of c5 (auto).
T=${1:-r2g}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "steps_parity or errors" > gpurun_out/pytest_rules_$T.log 2>&1; tail -n 2 gpurun_out/pytest_rules_$T.log
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d.get('ms_per_step'), d.get('parity',{}).get('match'), [ (k['kernel'], round(k['ms'],3)) for k in d['roofline']['kernels']])" $1 "$2" 2>&1 | tail -1; }
for p in 16 32; do
  for r in 2 3; do
    timeout 900 python bench.py --config c5 --p $p --cut-rule $r --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_c5_p${p}r${r}_$T.json 2> gpurun_out/bench_c5_p${p}r${r}_$T.err
    summ gpurun_out/bench_c5_p${p}r${r}_$T.json "c5 p=$p rule=$r"
  done
done
timeout 900 python tools/task_stats.py c5 16 auto > gpurun_out/tasks_c5_p16_$T.json 2> gpurun_out/tasks_c5_p16_$T.err
timeout 900 python tools/prof_paths.py run c2 c5 > gpurun_out/paths_$T.json 2> gpurun_out/paths_$T.err; cat gpurun_out/paths_$T.json
