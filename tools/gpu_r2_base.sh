mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2/pytest_gpu0.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2/pytest_gpu0.log
for c in cfg4 cfg5 cfg3; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2/bench0_$c.json 2> gpurun_out/r2/bench0_$c.err; done
