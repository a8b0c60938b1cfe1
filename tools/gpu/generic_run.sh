python -m pytest tests/test_generic_radius_gpu.py -x -q > gpurun_out/gen_tests.log 2>&1; echo rc=$? >> gpurun_out/gen_tests.log
python tools/prof_pass.py --radii 16,17,20,24,32,48,64,100 --shape 1,32768,32768 --reps 3 --tag generic >> gpurun_out/gen.jsonl 2>>gpurun_out/gen_err.log
python tools/prof_pass.py --radii 17,32,64 --shape 64,1024,1024 --reps 3 --tag generic64 >> gpurun_out/gen.jsonl 2>>gpurun_out/gen_err.log
python tools/prof_pass.py --mode exact --radii 17,32 --shape 64,1024,1024 --reps 3 --tag exact64 >> gpurun_out/gen.jsonl 2>>gpurun_out/gen_err.log
python -m pytest tests -m gpu -x -q > gpurun_out/gen_all_tests.log 2>&1; echo rc=$? >> gpurun_out/gen_all_tests.log
