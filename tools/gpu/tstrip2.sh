python -m pytest tests/test_exact_families_gpu.py tests/test_exact_gwalk_gpu.py tests/test_parity_gpu.py -q -x -m gpu 2>&1 | tail -2
rm -f gpurun_out/tstrip.jsonl
P="python tools/prof_pass.py --mode exact --reps 5"
$P --radii 2 --shape 64,1024,1024 --tag strips >> gpurun_out/tstrip.jsonl 2>gpurun_out/tstrip_err.log
$P --radii 2 --shape 1,4096,4096 --tag strips >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
$P --radii 2 --shape 1,4096,4096 --dtype u8 --tag strips >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
$P --radii 2 --shape 256,1024,1024 --tag strips >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
$P --radii 2 --shape 256,1024,1024 --dtype f32 --tag strips >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
$P --radii 3 --shape 3,1080,1920 --tag strips >> gpurun_out/tstrip.jsonl 2>>gpurun_out/tstrip_err.log
python -c "
import json
for l in open('gpurun_out/tstrip.jsonl'):
    d=json.loads(l); print(d['tag'],d['r'],d['shape'],d['dtype'],d['ms_per_pass'],d['kernel'])
"
tail -3 gpurun_out/tstrip_err.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tstrip_launches.csv python tools/prof_pass.py --mode exact --radii 2 --shape 64,1024,1024 --reps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tstrip_launches_c3.csv python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 2 > /dev/null 2>&1
