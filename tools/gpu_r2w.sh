#!/bin/bash
# Round 2 re-entry baseline: full GPU suite, smoke, default bench (c5), c2/c3/c4, per-vertex c2/c5.
T=${1:-r2w}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$T.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; tail -n 2 gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
timeout 900 python bench.py > gpurun_out/bench_default_$T.json 2> gpurun_out/bench_default_$T.err; cut -c1-300 gpurun_out/bench_default_$T.json
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d.get('ms_per_step'), d.get('parity',{}).get('match'), [ (k['kernel'], round(k['ms'],3)) for k in d['roofline']['kernels']])" $1 "$2" 2>&1 | tail -1; }
for c in c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_${c}_$T.json 2> gpurun_out/bench_${c}_$T.err
  summ gpurun_out/bench_${c}_$T.json $c
done
for c in c2 c5; do
  timeout 900 python bench.py --config $c --path vertex --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_vtx_${c}_$T.json 2> gpurun_out/bench_vtx_${c}_$T.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('vtx', sys.argv[2], d.get('ms_per_step'), d.get('parity'))" gpurun_out/bench_vtx_${c}_$T.json $c
done
