mkdir -p gpurun_out
for c in cfg4 cfg2 cfg5; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pass1_kernel -s 1 -c 1 -o gpurun_out/ncu_$c -f python tools/prof_solve.py $c > gpurun_out/ncu_$c.log 2>&1
done
