python -m pytest tests -m gpu -x -q > gpurun_out/disp_tests.log 2>&1; echo rc=$? >> gpurun_out/disp_tests.log
OSBF_GPU_EXACT=strip python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py -k "exact or c3" -x -q > gpurun_out/disp_strip_tests.log 2>&1; echo rc=$? >> gpurun_out/disp_strip_tests.log
