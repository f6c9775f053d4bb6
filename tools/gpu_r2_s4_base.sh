# session-4 baseline: GPU tests, smoke, cfg4 bench line
mkdir -p gpurun_out/s4
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/s4/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s4/bench_cfg4.json 2> gpurun_out/s4/bench_cfg4.err
