mkdir -p gpurun_out/s4
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s4/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/s4/pytest_gpu.log
for c in cfg3 cfg5 cfg1; do timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/s4/bench_$c.json 2>/dev/null; done
