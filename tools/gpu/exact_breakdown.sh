# Full GPU suite (no -x) + per-kernel times of the exact paths.
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_all.log
for cfg in "64,1024,1024 2,8,32" "1,4096,4096 2"; do
  set -- $cfg
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_launches_$1.csv \
    python tools/prof_pass.py --mode exact --radii $2 --shape $1 --reps 2 > gpurun_out/exact_launches_$1.log 2>&1
done
tail -3 gpurun_out/gpu_tests_all.log
