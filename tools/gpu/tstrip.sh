python -m pytest tests/test_exact_gwalk_gpu.py tests/test_exact_families_gpu.py tests/test_exact_twalk_gpu.py tests/test_parity_gpu.py tests/test_api_gpu.py tests/test_boxfilter.py tests/test_fastosbf_gpu.py tests/test_acceptance_gpu.py -q -x -m gpu > gpurun_out/tstrip_tests.log 2>&1; echo rc=$? >> gpurun_out/tstrip_tests.log
tail -5 gpurun_out/tstrip_tests.log
rm -f gpurun_out/tstrip.jsonl
P="python tools/prof_pass.py --mode exact --reps 5"
for fam in strips chains; do
OSBF_GPU_TABLE=$fam $P --radii 2,32 --shape 64,1024,1024 --tag $fam >> gpurun_out/tstrip.jsonl 2>gpurun_out/tstrip_err.log
OSBF_GPU_TABLE=$fam $P --radii 2 --shape 1,4096,4096 --tag $fam >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
OSBF_GPU_TABLE=$fam $P --radii 2 --shape 1,4096,4096 --dtype u8 --tag $fam >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
OSBF_GPU_TABLE=$fam $P --radii 2 --shape 256,1024,1024 --tag $fam >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
OSBF_GPU_TABLE=$fam $P --radii 2 --shape 256,1024,1024 --dtype f32 --tag $fam >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
OSBF_GPU_TABLE=$fam $P --radii 3 --shape 3,1080,1920 --tag $fam >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
OSBF_GPU_TABLE=$fam $P --radii 2 --shape 1,512,512 --tag $fam >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
OSBF_GPU_TABLE=$fam $P --radii 4 --shape 1,32768,32768 --tag $fam >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
OSBF_GPU_TABLE=$fam $P --radii 2 --shape 1000,128,128 --tag $fam >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
done
python -c "
import json
for l in open('gpurun_out/tstrip.jsonl'):
    d=json.loads(l); print(d['tag'],d['r'],d['shape'],d['dtype'],d['ms_per_pass'],d['kernel'])
"
tail -3 gpurun_out/tstrip_err.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tstrip_launches.csv python tools/prof_pass.py --mode exact --radii 2 --shape 64,1024,1024 --reps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tstrip_launches_c3.csv python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 2 > /dev/null 2>&1
tail -4 gpurun_out/tstrip_launches.csv | cut -c1-200; tail -4 gpurun_out/tstrip_launches_c3.csv | cut -c1-200
