python -m pytest tests/test_exact_gwalk_gpu.py tests/test_acceptance_gpu.py tests/test_exact_twalk_gpu.py tests/test_parity_gpu.py -q -x > gpurun_out/gwalk_tests.log 2>&1; echo rc=$? >> gpurun_out/gwalk_tests.log
tail -5 gpurun_out/gwalk_tests.log
rm -f gpurun_out/gwalk2.jsonl
P="python tools/prof_pass.py --mode exact --reps 5"
for deep in 0 1; do
OSBF_GPU_TABLE_DEEP=$deep $P --radii 32 --shape 64,1024,1024 --tag deep$deep >> gpurun_out/gwalk2.jsonl 2>gpurun_out/gwalk_err.log
OSBF_GPU_TABLE_DEEP=$deep $P --radii 32 --shape 256,1024,1024 --tag deep$deep >> gpurun_out/gwalk2.jsonl 2>>gpurun_out/gwalk_err.log
OSBF_GPU_TABLE_DEEP=$deep $P --radii 32 --shape 3,1080,1920 --tag deep$deep >> gpurun_out/gwalk2.jsonl 2>>gpurun_out/gwalk_err.log
OSBF_GPU_TABLE_DEEP=$deep $P --radii 32 --shape 1,512,512 --tag deep$deep >> gpurun_out/gwalk2.jsonl 2>>gpurun_out/gwalk_err.log
OSBF_GPU_TABLE_DEEP=$deep $P --radii 32 --shape 16,2048,2048 --tag deep$deep >> gpurun_out/gwalk2.jsonl 2>>gpurun_out/gwalk_err.log
OSBF_GPU_TABLE_DEEP=$deep OSBF_GPU_EXACT=table $P --radii 2,8,16 --shape 64,1024,1024 --tag table_deep$deep >> gpurun_out/gwalk2.jsonl 2>>gpurun_out/gwalk_err.log
OSBF_GPU_TABLE_DEEP=$deep OSBF_GPU_EXACT=table $P --radii 2 --shape 256,1024,1024 --tag table_deep$deep >> gpurun_out/gwalk2.jsonl 2>>gpurun_out/gwalk_err.log
done
$P --radii 2 --shape 256,1024,1024 --tag default >> gpurun_out/gwalk2.jsonl 2>>gpurun_out/gwalk_err.log
python -c "
import json
for l in open('gpurun_out/gwalk2.jsonl'):
    d=json.loads(l); print(d['tag'],d['r'],d['shape'],d['ms_per_pass'],d['kernel'])
"
tail -3 gpurun_out/gwalk_err.log
