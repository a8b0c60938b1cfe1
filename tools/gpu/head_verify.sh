# HEAD verification: GPU tests, bench line, fp64 latency probe.
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat_probe tools/probes/lat_probe.cu && /tmp/lat_probe > gpurun_out/lat_probe.txt 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/bench.err; cat gpurun_out/lat_probe.txt
