# round 2: bench lines for every config + the reference arm (cfg4)
mkdir -p gpurun_out/r2
for c in ${CFGS:-cfg4 cfg5 cfg3 cfg2 cfg1}; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2/bench_ref_cfg4.json 2> gpurun_out/r2/bench_ref_cfg4.err
nproc > gpurun_out/r2/nproc.txt
