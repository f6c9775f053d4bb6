mkdir -p gpurun_out
for c in cfg1; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
