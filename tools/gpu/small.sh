python tools/prof_pass.py --radii 3,4,6 --shape 3,1080,1920 --reps 20 --tag c2_walk >> gpurun_out/small.jsonl 2>>gpurun_out/small_err.log
OSBF_GPU_FAST=tma python tools/prof_pass.py --radii 3,4 --shape 3,1080,1920 --reps 20 --tag c2_tma >> gpurun_out/small.jsonl 2>>gpurun_out/small_err.log
OSBF_GPU_FAST=stream python tools/prof_pass.py --radii 6 --shape 3,1080,1920 --reps 20 --tag c2_stream >> gpurun_out/small.jsonl 2>>gpurun_out/small_err.log
python tools/prof_pass.py --radii 3,4 --shape 1,2048,2048 --reps 20 --tag s2k_walk >> gpurun_out/small.jsonl 2>>gpurun_out/small_err.log
OSBF_GPU_FAST=tma python tools/prof_pass.py --radii 3,4 --shape 1,2048,2048 --reps 20 --tag s2k_tma >> gpurun_out/small.jsonl 2>>gpurun_out/small_err.log
python tools/prof_pass.py --radii 3,4,8 --shape 1,1024,1024 --reps 20 --tag s1k_walk >> gpurun_out/small.jsonl 2>>gpurun_out/small_err.log
OSBF_GPU_FAST=tma python tools/prof_pass.py --radii 3,4 --shape 1,1024,1024 --reps 20 --tag s1k_tma >> gpurun_out/small.jsonl 2>>gpurun_out/small_err.log
