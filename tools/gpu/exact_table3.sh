OSBF_GPU_EXACT=table python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py tests/test_fastosbf_gpu.py tests/test_boxfilter.py tests/test_api_gpu.py -k "exact or c3 or C3 or sat or fast_osbf or box or means or sel or diag" -x -q > gpurun_out/ext3_tests.log 2>&1; echo rc=$? >> gpurun_out/ext3_tests.log
OSBF_GPU_EXACT=table python tools/prof_pass.py --mode exact --radii 1,2,4,8,16,32 --shape 1,4096,4096 --reps 10 --tag table >> gpurun_out/ext3.jsonl 2>>gpurun_out/ext3_err.log
OSBF_GPU_EXACT=table python tools/prof_pass.py --mode exact --radii 2,8,16 --shape 64,1024,1024 --reps 5 --tag table64 >> gpurun_out/ext3.jsonl 2>>gpurun_out/ext3_err.log
python tools/prof_pass.py --mode exact --radii 2,8,16 --shape 64,1024,1024 --reps 5 --tag fused64 >> gpurun_out/ext3.jsonl 2>>gpurun_out/ext3_err.log
python tools/prof_pass.py --mode exact --radii 2,16 --shape 1,1080,1920 --reps 10 --tag fusedC2 >> gpurun_out/ext3.jsonl 2>>gpurun_out/ext3_err.log
OSBF_GPU_EXACT=table python tools/prof_pass.py --mode exact --radii 2,16 --shape 1,1080,1920 --reps 10 --tag tableC2 >> gpurun_out/ext3.jsonl 2>>gpurun_out/ext3_err.log
OSBF_GPU_EXACT=table python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 3 > gpurun_out/ext3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ext3_launches.csv env OSBF_GPU_EXACT=table python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 3 > gpurun_out/ext3_ncu.log 2>&1
