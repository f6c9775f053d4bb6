mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:strip_kernel -s 1 -c 1 -o gpurun_out/ncu_strip_final -f python tools/prof_solve.py cfg4 > gpurun_out/ncu_strip_final.log 2>&1
for c in cfg4 cfg3 cfg5; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
