# Launch list of the default bench command (our kernels only) + timings of
# the other table-path users (box_filter, fast_osbf) after the strip builder.
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_short.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fast_|exact_|convert_|quarter|box|fastosbf|select" -c 900 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
python tools/prof_pass.py --mode box --radii 2,8 --shape 64,1024,1024 --reps 5 --tag box > gpurun_out/others.jsonl 2>/dev/null
python tools/prof_pass.py --mode fastosbf --radii 2,8 --shape 64,1024,1024 --reps 5 --tag fastosbf >> gpurun_out/others.jsonl 2>/dev/null
python tools/prof_pass.py --mode box --radii 4 --shape 1,4096,4096 --reps 5 --tag box >> gpurun_out/others.jsonl 2>/dev/null
python tools/prof_pass.py --mode fastosbf --radii 4 --shape 1,4096,4096 --reps 5 --tag fastosbf >> gpurun_out/others.jsonl 2>/dev/null
cat gpurun_out/others.jsonl | cut -c1-220
