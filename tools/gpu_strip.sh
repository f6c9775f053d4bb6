mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "seed or cfg4 or cfg5" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/time_cfg4.py > gpurun_out/time_cfg4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_seed.csv python tools/prof_solve.py cfg4 > /dev/null 2>&1
