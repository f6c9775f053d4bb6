mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "strip or wide or cfg4" > gpurun_out/pytest_strip.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_strip.log
timeout 300 python tools/time_cfg4.py > gpurun_out/time_cfg4.log 2>&1
