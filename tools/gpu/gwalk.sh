python -m pytest tests/test_exact_gwalk_gpu.py tests/test_acceptance_gpu.py tests/test_generic_radius_gpu.py -q > gpurun_out/gwalk_tests.log 2>&1; echo rc=$? >> gpurun_out/gwalk_tests.log
tail -15 gpurun_out/gwalk_tests.log
rm -f gpurun_out/gwalk.jsonl
python tools/prof_pass.py --mode exact --radii 2,8,17,32,62 --shape 64,1024,1024 --reps 5 --tag gwalk >> gpurun_out/gwalk.jsonl 2>gpurun_out/gwalk_err.log
OSBF_GPU_GWALK=0 python tools/prof_pass.py --mode exact --radii 17,32,62 --shape 64,1024,1024 --reps 5 --tag stencil >> gpurun_out/gwalk.jsonl 2>>gpurun_out/gwalk_err.log
OSBF_GPU_TABLE_DEEP=1 python tools/prof_pass.py --mode exact --radii 17,32 --shape 64,1024,1024 --reps 5 --tag gwalk_deep >> gpurun_out/gwalk.jsonl 2>>gpurun_out/gwalk_err.log
OSBF_GPU_GWALK_STAGES=2 python tools/prof_pass.py --mode exact --radii 17,32,62 --shape 64,1024,1024 --reps 5 --tag gwalk_ns2 >> gpurun_out/gwalk.jsonl 2>>gpurun_out/gwalk_err.log
OSBF_GPU_GWALK_STAGES=4 python tools/prof_pass.py --mode exact --radii 17,32 --shape 64,1024,1024 --reps 5 --tag gwalk_ns4 >> gpurun_out/gwalk.jsonl 2>>gpurun_out/gwalk_err.log
python tools/prof_pass.py --mode exact --radii 16,17,32 --shape 1,4096,4096 --reps 5 --tag gwalk_c3 >> gpurun_out/gwalk.jsonl 2>>gpurun_out/gwalk_err.log
OSBF_GPU_GWALK=0 python tools/prof_pass.py --mode exact --radii 17,32 --shape 1,4096,4096 --reps 5 --tag stencil_c3 >> gpurun_out/gwalk.jsonl 2>>gpurun_out/gwalk_err.log
cat gpurun_out/gwalk.jsonl | cut -c1-260
tail -3 gpurun_out/gwalk_err.log
