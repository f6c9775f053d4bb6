mkdir -p gpurun_out
timeout 900 python tools/time_next_rows.py > gpurun_out/next_rows.log 2>&1
