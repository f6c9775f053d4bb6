# round 2 campaign: GPU tests, smoke, every bench line, the reference arm, the cfg4
# bench launch list, the one-GPU rank emulation
mkdir -p gpurun_out/r2/final
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv > gpurun_out/r2/final/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2/final/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2/final/smoke.log 2>&1
for c in cfg4 cfg5 cfg3 cfg2 cfg1 cfg4_p99 cfg4_planted; do
  timeout 600 python bench.py --config $c > gpurun_out/r2/final/bench_$c.json 2> gpurun_out/r2/final/bench_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/r2/final/bench_ref_cfg4.json 2> gpurun_out/r2/final/bench_ref_cfg4.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2/final/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-verify --e2e-steps 1 > gpurun_out/r2/final/ncu_launch.log 2>&1
python tools/rank_emulation.py cfg4 > gpurun_out/r2/final/rank_emu_cfg4.jsonl 2>&1
python tools/rank_emulation.py cfg5 > gpurun_out/r2/final/rank_emu_cfg5.jsonl 2>&1
nproc > gpurun_out/r2/final/nproc.txt
