#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_c2_ws2.json 2> gpurun_out/bench_c2_ws2.err
echo "torchrun rc=$?"; tail -3 gpurun_out/bench_c2_ws2.err; cut -c1-600 gpurun_out/bench_c2_ws2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5v2.csv \
    python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_c5v2_ncu.json 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_tc_rows -s 1 -c 1 -o gpurun_out/prof_c5v2 -f \
    python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_c5v2.log 2>&1
tail -2 gpurun_out/ncu_full_c5v2.log
