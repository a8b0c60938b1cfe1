python -m pytest tests -m gpu -x -q > gpurun_out/walk2_tests.log 2>&1; echo rc=$? >> gpurun_out/walk2_tests.log
for band in 512 1024 2048; do
  OSBF_GPU_WALK_BAND=$band python tools/prof_pass.py --radii 3,4,5,6,8,12,16 --shape 1,32768,32768 --reps 5 --tag walk_b$band >> gpurun_out/walk2_c5.jsonl 2>>gpurun_out/walk2_err.log
done
python tools/prof_pass.py --radii 1,2,3,4,5,6,8,12,16 --shape 256,1024,1024 --reps 5 --tag default >> gpurun_out/walk2_c4.jsonl 2>>gpurun_out/walk2_err.log
