python -m pytest tests/test_fast_families_gpu.py -k "walk" -x -q > gpurun_out/w56_tests.log 2>&1; echo rc=$? >> gpurun_out/w56_tests.log
python tools/prof_pass.py --radii 4,5,6,7,8 --shape 1,32768,32768 --reps 5 --tag w56 >> gpurun_out/w56.jsonl 2>>gpurun_out/w56_err.log
python tools/prof_pass.py --radii 5,6 --shape 256,1024,1024 --reps 5 --tag w56c4 >> gpurun_out/w56.jsonl 2>>gpurun_out/w56_err.log
