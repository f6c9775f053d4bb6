mkdir -p gpurun_out
MSQ_TEST_FLOOR=133 timeout 600 ncu --set full --clock-control none --import-source on -k regex:strip_kernel -s 1 -c 1 -o gpurun_out/ncu_strip133 -f python tools/prof_solve.py cfg4 > gpurun_out/ncu_strip133.log 2>&1
