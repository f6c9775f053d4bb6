mkdir -p gpurun_out
timeout 600 python tools/time_pack.py > gpurun_out/time_pack.log 2>&1
