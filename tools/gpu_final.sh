#!/bin/bash
# Round-end measurement: GPU tests, smoke, default bench line + ncu (c2), the other
# configs' lines, c5s ncu, NEXT-row paths, and the N>1 flow (2 ranks, gloo on one GPU).
T=${1:-f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$T.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; tail -n 2 gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
timeout 600 python bench.py > gpurun_out/bench_default_$T.json 2> gpurun_out/bench_default_$T.err; cut -c1-200 gpurun_out/bench_default_$T.json
bash tools/gpu_bench_profile.sh c2 c2$T > /dev/null 2>&1
for c in c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c$T.json 2> gpurun_out/bench_$c$T.err
  cut -c1-160 gpurun_out/bench_$c$T.json
done
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_tc_(rows|light)" -s 2 -c 2 -o gpurun_out/prof_c5s$T -f python bench.py --config c5s --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_c5s$T.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_tc_(rows|light)" -s 2 -c 2 -o gpurun_out/prof_c3$T -f python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_c3$T.log 2>&1
for c in c2 c5; do
  timeout 900 python bench.py --config $c --path vertex --steps 3 --warmup 2 > gpurun_out/bench_vtx_$c$T.json 2> gpurun_out/bench_vtx_$c$T.err
  timeout 900 python bench.py --config $c --path cc --steps 3 --warmup 1 > gpurun_out/bench_cc_$c$T.json 2> gpurun_out/bench_cc_$c$T.err
done
timeout 900 python bench.py --config c5 --budget-gb 12 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c5b12$T.json 2> gpurun_out/bench_c5b12$T.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_ws2$T.json 2> gpurun_out/bench_ws2$T.err; echo "ws2 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref$T.json 2> gpurun_out/ref$T.err; cut -c1-160 gpurun_out/ref$T.json
timeout 1500 python tools/sim_ranks.py c5 1 2 4 8 --measured > gpurun_out/simm_c5$T.json 2> gpurun_out/simm_c5$T.err; tail -n 1 gpurun_out/simm_c5$T.err
