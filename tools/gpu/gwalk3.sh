rm -f gpurun_out/gwalk3.jsonl
P="python tools/prof_pass.py --mode exact --reps 5"
for tw in 1 0; do
OSBF_GPU_TWALK=$tw OSBF_GPU_EXACT=table $P --radii 1,2,4,8,16 --shape 64,1024,1024 --tag twalk$tw >> gpurun_out/gwalk3.jsonl 2>gpurun_out/gwalk_err.log
OSBF_GPU_TWALK=$tw OSBF_GPU_EXACT=table $P --radii 1,2,4,8,16 --shape 1,4096,4096 --tag twalk$tw >> gpurun_out/gwalk3.jsonl 2>>gpurun_out/gwalk_err.log
OSBF_GPU_TWALK=$tw OSBF_GPU_EXACT=table $P --radii 2 --shape 256,1024,1024 --tag twalk$tw >> gpurun_out/gwalk3.jsonl 2>>gpurun_out/gwalk_err.log
OSBF_GPU_TWALK=$tw OSBF_GPU_EXACT=table $P --radii 3 --shape 3,1080,1920 --tag twalk$tw >> gpurun_out/gwalk3.jsonl 2>>gpurun_out/gwalk_err.log
OSBF_GPU_TWALK=$tw OSBF_GPU_EXACT=table $P --radii 2 --shape 1,512,512 --tag twalk$tw >> gpurun_out/gwalk3.jsonl 2>>gpurun_out/gwalk_err.log
done
$P --radii 1,2 --shape 1,512,512 --tag default >> gpurun_out/gwalk3.jsonl 2>>gpurun_out/gwalk_err.log
$P --radii 3 --shape 3,1080,1920 --tag default >> gpurun_out/gwalk3.jsonl 2>>gpurun_out/gwalk_err.log
$P --radii 1 --shape 64,1024,1024 --tag default >> gpurun_out/gwalk3.jsonl 2>>gpurun_out/gwalk_err.log
python -c "
import json
for l in open('gpurun_out/gwalk3.jsonl'):
    d=json.loads(l); print(d['tag'],d['r'],d['shape'],d['ms_per_pass'],d['kernel'])
"
tail -3 gpurun_out/gwalk_err.log
