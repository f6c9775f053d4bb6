mkdir -p gpurun_out/s4
timeout 1200 python -m pytest tests/test_gpu_sieve.py tests/test_capi.py -q -x > gpurun_out/s4/pytest_sieve.log 2>&1; echo "rc=$?" >> gpurun_out/s4/pytest_sieve.log
python tools/rank_emulation.py cfg4 > gpurun_out/s4/rank_emu_cfg4_sieve.jsonl 2>&1
python tools/rank_emulation.py cfg4 band > gpurun_out/s4/rank_emu_cfg4_band.jsonl 2>&1
