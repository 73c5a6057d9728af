mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r2a.log 2>&1; tail -n 3 gpurun_out/pytest_gpu_r2a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
timeout 900 python bench.py > gpurun_out/bench_default_r2a.json 2> gpurun_out/bench_default_r2a.err; cut -c1-400 gpurun_out/bench_default_r2a.json; tail -3 gpurun_out/bench_default_r2a.err
bash tools/gpu_r2_probe.sh r2a
