# sieve engine: random cases, then one ncu --set full capture of the 3 sieve kernels (2nd solve of cfg4)
mkdir -p gpurun_out/s4
timeout 600 python tools/sieve_check.py quick > gpurun_out/s4/sieve_quick.log 2>&1; echo "rc=$?" >> gpurun_out/s4/sieve_quick.log
timeout 300 python tools/sieve_check.py cfg4 ${WPC:-5} > gpurun_out/s4/sieve_cfg4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve -s 3 -c 3 -o /tmp/cap_sieve -f python tools/prof_solve.py cfg4 > gpurun_out/s4/ncu_sieve.log 2>&1
ncu -i /tmp/cap_sieve.ncu-rep --page details --csv > gpurun_out/s4/sieve_details.csv 2>&1
ncu -i /tmp/cap_sieve.ncu-rep --page source --csv --kernel-name regex:sieve_pass > gpurun_out/s4/sieve_pass_source.csv 2>&1
ncu -i /tmp/cap_sieve.ncu-rep --page source --csv --kernel-name regex:sieve_verify > gpurun_out/s4/sieve_verify_source.csv 2>&1
ncu -i /tmp/cap_sieve.ncu-rep --page source --csv --kernel-name regex:sieve_edge > gpurun_out/s4/sieve_edge_source.csv 2>&1
