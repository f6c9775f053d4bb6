# session-4: GPU tests, smoke, bench lines
mkdir -p gpurun_out/s4
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s4/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/s4/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4/smoke.log 2>&1
for c in ${CFGS:-cfg4 cfg4_p99 cfg4_planted}; do
  timeout 600 python bench.py --config $c > gpurun_out/s4/bench_$c.json 2> gpurun_out/s4/bench_$c.err
done
