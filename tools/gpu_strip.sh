mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/time_small.py > gpurun_out/time_small.log 2>&1
timeout 300 python bench.py --config cfg1 --steps 30 --warmup 5 > gpurun_out/bench_cfg1.json 2>gpurun_out/bench_cfg1.err
