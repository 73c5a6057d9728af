#!/bin/bash
# Round 2: bit-sliced hit counters for the per-vertex dense pairs -- parity, vertex timings vs the previous path.
T=${1:-r2ag}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_vertex.py -q -x -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1; tail -n 2 gpurun_out/pytest_$T.log
for v in "" noslice; do
  for c in c2 c5s c5; do
    PGABB_LIB_VARIANT=$v timeout 900 python bench.py --config $c --path vertex --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_vtx_${c}_$T$v.json 2> gpurun_out/bench_vtx_${c}_$T$v.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('vtx', sys.argv[2], d.get('ms_per_step'), d.get('parity',{}).get('match'), [(k['kernel'], round(k['ms'],2)) for k in d['roofline']['kernels']])" gpurun_out/bench_vtx_${c}_$T$v.json "$c ${v:-sliced}"
  done
done
timeout 900 python tools/prof_paths.py run c2:vertex c5s:vertex > gpurun_out/paths_$T.json 2> gpurun_out/paths_$T.err
cat gpurun_out/paths_$T.json; tail -2 gpurun_out/paths_$T.err
