python -m pytest tests/test_filters3d.py tests/test_acceptance_gpu.py -k "3d or 3D or volume or criterion8 or svt" -x -q > gpurun_out/f3d_tests.log 2>&1; echo rc=$? >> gpurun_out/f3d_tests.log
python tools/prof_pass.py --mode osbf3d --radii 1,2,4,8,12 --shape 256,256,256 --reps 5 --tag osbf3d >> gpurun_out/f3d.jsonl 2>>gpurun_out/f3d_err.log
python tools/prof_pass.py --mode box3d --radii 2,8 --shape 256,256,256 --reps 5 --tag box3d >> gpurun_out/f3d.jsonl 2>>gpurun_out/f3d_err.log
