# sieve engine: random cases vs the oracle, cfg4 timing for a few CTA shapes
mkdir -p gpurun_out/s4
timeout 600 python tools/sieve_check.py quick > gpurun_out/s4/sieve_quick.log 2>&1; echo "rc=$?" >> gpurun_out/s4/sieve_quick.log
for w in ${WPCS:-3 5}; do
timeout 300 python tools/sieve_check.py cfg4 $w > gpurun_out/s4/sieve_cfg4_w$w.log 2>&1; echo "rc=$?" >> gpurun_out/s4/sieve_cfg4_w$w.log
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sieve -c 12 --csv --log-file gpurun_out/s4/sieve_launches.csv python tools/prof_solve.py cfg4 > gpurun_out/s4/sieve_launch.log 2>&1
