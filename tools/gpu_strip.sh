mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_histogram_gpu.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/time_next_rows.py > gpurun_out/next_rows.log 2>&1
