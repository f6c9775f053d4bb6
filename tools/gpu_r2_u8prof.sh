# round 2: launch lists + ncu full captures of the u8 band pass (cfg5, cfg3); reports exported on the box
mkdir -p gpurun_out/r2
for c in cfg5 cfg3; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2/launches_$c.csv python tools/prof_solve.py $c > gpurun_out/r2/launch_$c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pass1_kernel -s 1 -c 1 -o /tmp/ncu_pass1_$c -f python tools/prof_solve.py $c > gpurun_out/r2/ncu_$c.log 2>&1
ncu -i /tmp/ncu_pass1_$c.ncu-rep --page details --csv > gpurun_out/r2/ncu_pass1_${c}_details.csv 2>&1
ncu -i /tmp/ncu_pass1_$c.ncu-rep --page raw --csv > gpurun_out/r2/ncu_pass1_${c}_raw.csv 2>&1
ncu -i /tmp/ncu_pass1_$c.ncu-rep --page source --csv --print-source cuda > gpurun_out/r2/ncu_pass1_${c}_source.csv 2>&1
ls -la /tmp/ncu_pass1_$c.ncu-rep >> gpurun_out/r2/ncu_$c.log
done
du -sh gpurun_out
