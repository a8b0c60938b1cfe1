true
true
rm -f gpurun_out/gw4.jsonl
P="python tools/prof_pass.py --mode exact --reps 5"
$P --radii 2,32 --shape 64,1024,1024 --tag gw4 >> gpurun_out/gw4.jsonl 2>gpurun_out/gw4_err.log
$P --radii 2,16 --shape 1,4096,4096 --tag gw4 >> gpurun_out/gw4.jsonl 2>>gpurun_out/gw4_err.log
$P --radii 2 --shape 256,1024,1024 --tag gw4 >> gpurun_out/gw4.jsonl 2>>gpurun_out/gw4_err.log
python -c "
import json
for l in open('gpurun_out/gw4.jsonl'):
    d=json.loads(l); print(d['tag'],d['r'],d['shape'],d['ms_per_pass'],d['kernel'])
"
tail -2 gpurun_out/gw4_err.log
