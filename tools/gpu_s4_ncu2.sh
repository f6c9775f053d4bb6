mkdir -p gpurun_out/s4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sieve_(coarse|verify)" -s 2 -c 2 -o /tmp/cap_sieve2 -f python tools/prof_solve.py cfg4 > gpurun_out/s4/ncu_sieve2.log 2>&1
ncu -i /tmp/cap_sieve2.ncu-rep --page details --csv > gpurun_out/s4/sieve2_details.csv 2>&1
ncu -i /tmp/cap_sieve2.ncu-rep --page source --csv --kernel-name regex:sieve_coarse > gpurun_out/s4/sieve_coarse_source.csv 2>&1
ncu -i /tmp/cap_sieve2.ncu-rep --page source --csv --kernel-name regex:sieve_verify > gpurun_out/s4/sieve_verify_source.csv 2>&1
