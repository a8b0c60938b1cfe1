python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py -k "exact or c3 or C3 or sat or nonfinite or nan or inf" -x -q > gpurun_out/ext4_tests.log 2>&1; echo rc=$? >> gpurun_out/ext4_tests.log
python tools/prof_pass.py --mode exact --radii 1,2,4,8,16,32 --shape 1,4096,4096 --reps 10 --tag table >> gpurun_out/ext4.jsonl 2>>gpurun_out/ext4_err.log
python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 3 > gpurun_out/ext4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"col_chain_deep|exact_stencil" -s 2 -c 2 -o gpurun_out/deep4 python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 3 > gpurun_out/ext4_ncu.log 2>&1
