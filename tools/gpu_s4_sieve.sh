# sieve engine: random cases vs the oracle, cfg4 timing
mkdir -p gpurun_out/s4
timeout 600 python tools/sieve_check.py quick > gpurun_out/s4/sieve_quick.log 2>&1; echo "rc=$?" >> gpurun_out/s4/sieve_quick.log
for w in 3 2 5; do
timeout 300 python tools/sieve_check.py cfg4 $w > gpurun_out/s4/sieve_cfg4_w$w.log 2>&1; echo "rc=$?" >> gpurun_out/s4/sieve_cfg4_w$w.log
done
