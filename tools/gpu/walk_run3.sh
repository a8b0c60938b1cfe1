python -m pytest tests/test_parity_gpu.py tests/test_fast_families_gpu.py -x -q > gpurun_out/walk3_tests.log 2>&1; echo rc=$? >> gpurun_out/walk3_tests.log
python tools/prof_pass.py --radii 1,2,3,4,6,8,12,16 --shape 1,4096,4096 --reps 20 --tag c3shape >> gpurun_out/walk3.jsonl 2>>gpurun_out/walk3_err.log
OSBF_GPU_FAST=tma python tools/prof_pass.py --radii 3,4 --shape 1,4096,4096 --reps 20 --tag c3shape_tma >> gpurun_out/walk3.jsonl 2>>gpurun_out/walk3_err.log
OSBF_GPU_FAST=stream python tools/prof_pass.py --radii 6,8,12,16 --shape 1,4096,4096 --reps 20 --tag c3shape_stream >> gpurun_out/walk3.jsonl 2>>gpurun_out/walk3_err.log
