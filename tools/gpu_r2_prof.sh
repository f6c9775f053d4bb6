# round 2: launch lists (repo kernels only) + one ncu --set full capture of a kernel
mkdir -p gpurun_out/r2
K=${KERN:-ustrip_kernel}
for c in ${CFGS:-cfg3}; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:strip|pass1|seed|carry|fixup|team" -c 12 --csv --log-file gpurun_out/r2/pf_launches_$c.csv python tools/prof_solve.py $c > gpurun_out/r2/pf_launch_$c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o /tmp/pf_$c -f python tools/prof_solve.py $c > gpurun_out/r2/pf_ncu_$c.log 2>&1
ncu -i /tmp/pf_$c.ncu-rep --page details --csv > gpurun_out/r2/pf_${c}_details.csv 2>&1
ncu -i /tmp/pf_$c.ncu-rep --page raw --csv > gpurun_out/r2/pf_${c}_raw.csv 2>&1
ncu -i /tmp/pf_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/r2/pf_${c}_sass.csv 2>&1
done
