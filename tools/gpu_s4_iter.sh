mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests/test_gpu_sieve.py tests/test_capi.py -q -x > gpurun_out/s4/pytest_sieve.log 2>&1; echo "rc=$?" >> gpurun_out/s4/pytest_sieve.log
timeout 300 python tools/sieve_check.py cfg4 > gpurun_out/s4/sieve_cfg4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sieve -c 12 --csv --log-file gpurun_out/s4/sieve_launches.csv python tools/prof_solve.py cfg4 > gpurun_out/s4/sieve_launch.log 2>&1
