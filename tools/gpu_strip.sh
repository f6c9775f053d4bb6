mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cfg4 or band or ranks or team" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/time_cfg4.py > gpurun_out/time_cfg4.log 2>&1
timeout 300 python tools/time_small.py > gpurun_out/time_small.log 2>&1
