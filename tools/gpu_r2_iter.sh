# round 2 iteration: GPU tests, u8 bench lines, msq launch lists
mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/r2/it_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2/it_pytest.log
for c in ${CFGS:-cfg5 cfg3}; do
timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2/it_bench_$c.json 2> gpurun_out/r2/it_bench_$c.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:msq -c 12 --csv --log-file gpurun_out/r2/it_launches_$c.csv python tools/prof_solve.py $c > gpurun_out/r2/it_launch_$c.log 2>&1
done
