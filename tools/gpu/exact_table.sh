OSBF_GPU_EXACT=table python -m pytest tests/test_parity_gpu.py -k "exact or c3 or C3 or sat" -x -q > gpurun_out/ext_tests.log 2>&1; echo rc=$? >> gpurun_out/ext_tests.log
python -m pytest tests/test_configs_gpu.py -k c3 -x -q >> gpurun_out/ext_tests.log 2>&1; echo rc=$? >> gpurun_out/ext_tests.log
OSBF_GPU_EXACT=table python tools/prof_pass.py --mode exact --radii 1,2,4,8,16 --shape 1,4096,4096 --reps 10 --tag table >> gpurun_out/ext.jsonl 2>>gpurun_out/ext_err.log
python tools/prof_pass.py --mode exact --radii 2,8 --shape 1,4096,4096 --reps 10 --tag fused >> gpurun_out/ext.jsonl 2>>gpurun_out/ext_err.log
OSBF_GPU_EXACT=table python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 3 > gpurun_out/ext_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ext_launches.csv env OSBF_GPU_EXACT=table python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 3 > gpurun_out/ext_ncu.log 2>&1
