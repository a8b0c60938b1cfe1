python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_all.log
tail -4 gpurun_out/gpu_tests_all.log
rm -f gpurun_out/exact_paths.jsonl
P="python tools/prof_pass.py --mode exact --reps 5"
for fam in gwalk strip; do
OSBF_GPU_EXACT=$fam $P --radii 4 --shape 1,32768,32768 --dtype f32 --tag $fam >> gpurun_out/exact_paths.jsonl 2>gpurun_out/exact_paths_err.log
OSBF_GPU_EXACT=$fam $P --radii 2 --shape 1,1024,1024 --tag $fam >> gpurun_out/exact_paths.jsonl 2>>gpurun_out/exact_paths_err.log
OSBF_GPU_EXACT=$fam $P --radii 2 --shape 1000,128,128 --tag $fam >> gpurun_out/exact_paths.jsonl 2>>gpurun_out/exact_paths_err.log
OSBF_GPU_EXACT=$fam $P --radii 2 --shape 256,1024,1024 --dtype f32 --tag $fam >> gpurun_out/exact_paths.jsonl 2>>gpurun_out/exact_paths_err.log
done
python -c "
import json
for l in open('gpurun_out/exact_paths.jsonl'):
    d=json.loads(l); print(d['tag'],d['r'],d['shape'],d['dtype'],d['ms_per_pass'],d['kernel'])
"
tail -3 gpurun_out/exact_paths_err.log
