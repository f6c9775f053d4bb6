# stability: the GPU suite three times, the sieve tests ten times
mkdir -p gpurun_out/s4
for i in 1 2 3; do timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s4/flaky_all_$i.log 2>&1; echo "rc=$?" >> gpurun_out/s4/flaky_all_$i.log; done
for i in 1 2 3 4 5 6 7 8 9 10; do timeout 600 python -m pytest tests/test_gpu_sieve.py -q -x -p no:cacheprovider > gpurun_out/s4/flaky_sieve_$i.log 2>&1; echo "rc=$?" >> gpurun_out/s4/flaky_sieve_$i.log; done
