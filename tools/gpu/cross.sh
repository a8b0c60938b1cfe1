rm -f gpurun_out/cross.jsonl
python tools/prof_pass.py --mode exact --radii 17,20,24,32,48,62 --shape 1,32768,32768 --reps 3 --tag exact >> gpurun_out/cross.jsonl 2>gpurun_out/cross_err.log
python tools/prof_pass.py --mode fast --radii 17,20,24,32,48,56 --shape 1,32768,32768 --reps 3 --tag fast >> gpurun_out/cross.jsonl 2>>gpurun_out/cross_err.log
python tools/prof_pass.py --mode exact --radii 17,24,32 --shape 256,1024,1024 --reps 3 --tag exact >> gpurun_out/cross.jsonl 2>>gpurun_out/cross_err.log
python tools/prof_pass.py --mode fast --radii 17,24,32 --shape 256,1024,1024 --reps 3 --tag fast >> gpurun_out/cross.jsonl 2>>gpurun_out/cross_err.log
python tools/prof_pass.py --mode exact --radii 17,24,32 --shape 1,4096,4096 --reps 3 --tag exact >> gpurun_out/cross.jsonl 2>>gpurun_out/cross_err.log
python tools/prof_pass.py --mode fast --radii 17,24,32 --shape 1,4096,4096 --reps 3 --tag fast >> gpurun_out/cross.jsonl 2>>gpurun_out/cross_err.log
python -c "
import json
for l in open('gpurun_out/cross.jsonl'):
    d=json.loads(l); print(d['tag'],d['r'],d['shape'],d['ms_per_pass'],d['kernel'])
"
tail -2 gpurun_out/cross_err.log
