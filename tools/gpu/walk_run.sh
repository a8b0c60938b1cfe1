set -x
python -m pytest tests/test_fast_families_gpu.py -k "walk" -x -q > gpurun_out/walk_tests.log 2>&1; echo rc=$? >> gpurun_out/walk_tests.log
for fam in walk default; do
  if [ $fam = default ]; then unset OSBF_GPU_FAST; else export OSBF_GPU_FAST=$fam; fi
  python tools/prof_pass.py --radii 1,2,3,4,5,6,8,12,16 --shape 1,32768,32768 --reps 5 --tag $fam >> gpurun_out/walk_c5.jsonl 2>>gpurun_out/walk_err.log
  python tools/prof_pass.py --radii 1,2,4,8,16 --shape 256,1024,1024 --reps 5 --tag $fam >> gpurun_out/walk_c4.jsonl 2>>gpurun_out/walk_err.log
done
