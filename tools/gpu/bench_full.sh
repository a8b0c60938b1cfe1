# the driver's bench command, then the launch list of a short run of the same workload
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$? >> gpurun_out/bench_full.err
python bench.py --steps 1 --warmup 3 --no-sub --no-e2e --no-cpu-baseline > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_C5.csv python bench.py --steps 1 --warmup 3 --no-sub --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo rc=$? >> gpurun_out/bench_full.err
