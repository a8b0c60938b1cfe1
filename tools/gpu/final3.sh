python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_all.log
tail -3 gpurun_out/gpu_tests_all.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
python __graft_entry__.py smoke 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_launches_b64.csv python tools/prof_pass.py --mode exact --radii 2 --shape 64,1024,1024 --reps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exact_launches_c3.csv python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 2 > /dev/null 2>&1
for k in exact_table_strip exact_row_carries_pipe; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -f -o /tmp/rep_$k python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 1 > gpurun_out/ncu_$k.log 2>&1
python tools/ncu_top.py /tmp/rep_$k.ncu-rep 25 > gpurun_out/ncu_c3_$k.txt 2>&1
ncu -i /tmp/rep_$k.ncu-rep --page details > gpurun_out/ncu_c3_${k}_details.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -f -o /tmp/rep64_$k python tools/prof_pass.py --mode exact --radii 2 --shape 64,1024,1024 --reps 1 > gpurun_out/ncu64_$k.log 2>&1
python tools/ncu_top.py /tmp/rep64_$k.ncu-rep 25 > gpurun_out/ncu_b64_$k.txt 2>&1
ncu -i /tmp/rep64_$k.ncu-rep --page details > gpurun_out/ncu_b64_${k}_details.txt 2>&1
done
python tools/prof_pass.py --mode exact --radii 1,2,4,8,16,32,62 --shape 64,1024,1024 --reps 5 --tag final > gpurun_out/final_exact.jsonl 2>/dev/null
python tools/prof_pass.py --mode exact --radii 2 --shape 256,1024,1024 --dtype f32 --reps 5 --tag final_c4_first_pass >> gpurun_out/final_exact.jsonl 2>/dev/null
python tools/prof_pass.py --mode exact --radii 2 --shape 256,1024,1024 --reps 5 --tag final_c4 >> gpurun_out/final_exact.jsonl 2>/dev/null
python tools/prof_pass.py --mode exact --radii 4 --shape 1,32768,32768 --reps 3 --tag final_c5 >> gpurun_out/final_exact.jsonl 2>/dev/null
python tools/prof_pass.py --mode exact --radii 1,2,4,8,16,32 --shape 1,4096,4096 --reps 5 --tag final_c3 >> gpurun_out/final_exact.jsonl 2>/dev/null
