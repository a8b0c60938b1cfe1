python -m pytest tests/test_generic_radius_gpu.py tests/test_api_gpu.py -x -q > gpurun_out/gen2_tests.log 2>&1; echo rc=$? >> gpurun_out/gen2_tests.log
python tools/prof_pass.py --radii 17,20,24,32,48,64 --shape 1,32768,32768 --reps 3 --tag generic >> gpurun_out/gen2.jsonl 2>>gpurun_out/gen2_err.log
python tools/prof_pass.py --radii 17,32,64 --shape 64,1024,1024 --reps 3 --tag generic64 >> gpurun_out/gen2.jsonl 2>>gpurun_out/gen2_err.log
