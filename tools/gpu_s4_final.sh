# session-4 final campaign: GPU tests, smoke, every bench line, the reference arm, launch list of the
# bench command, ncu --set full of the sieve kernels, rank emulation, kernel-family check
O=gpurun_out/s4/final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv > $O/smi.txt
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for c in cfg4 cfg5 cfg3 cfg2 cfg1 cfg4_p99 cfg4_planted; do
  timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference > $O/bench_ref_cfg4.json 2> $O/bench_ref_cfg4.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg4_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-verify --e2e-steps 1 > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve -s 3 -c 3 -o /tmp/cap_sieve -f python tools/prof_solve.py cfg4 > $O/ncu_sieve.log 2>&1
ncu -i /tmp/cap_sieve.ncu-rep --page details --csv > $O/sieve_details.csv 2>&1
ncu -i /tmp/cap_sieve.ncu-rep --page source --csv --kernel-name regex:sieve_pass > $O/sieve_pass_source.csv 2>&1
python tools/rank_emulation.py cfg4 > $O/rank_emu_cfg4_sieve.jsonl 2>&1
python tools/rank_emulation.py cfg4 band > $O/rank_emu_cfg4_band.jsonl 2>&1
python tools/rank_emulation.py cfg5 > $O/rank_emu_cfg5.jsonl 2>&1
timeout 600 python tools/sanitize.py > $O/kernel_families.log 2>&1
nproc > $O/nproc.txt
