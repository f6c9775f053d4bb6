mkdir -p gpurun_out
for a in 0 1 2 3 7; do
  MSQ_NVCC_EXTRA="-DMSQ_STRIP_ABLATE=$a" python -c "from paper_2503_18974_b200 import build; build.build(force=True)" > /dev/null 2>&1
  echo "ablate=$a" >> gpurun_out/ablate.log
  MSQ_TEST_FLOOR=133 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:strip -c 3 --csv python tools/prof_solve.py cfg4 2>/dev/null | grep strip | tail -1 >> gpurun_out/ablate.log
done
