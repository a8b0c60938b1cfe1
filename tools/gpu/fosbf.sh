python -m pytest tests/test_fastosbf_gpu.py -x -q > gpurun_out/fosbf_tests.log 2>&1; echo rc=$? >> gpurun_out/fosbf_tests.log
python tools/prof_pass.py --mode fastosbf --radii 2,8 --shape 1,4096,4096 --reps 10 --tag fosbf_1 >> gpurun_out/fosbf.jsonl 2>>gpurun_out/fosbf_err.log
python tools/prof_pass.py --mode fastosbf --radii 2,8 --shape 256,1024,1024 --reps 3 --tag fosbf_256 >> gpurun_out/fosbf.jsonl 2>>gpurun_out/fosbf_err.log
