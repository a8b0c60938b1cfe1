python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_all.log
tail -4 gpurun_out/gpu_tests_all.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
