# ncu --set full of the exact table-path kernels; reports stay on the box
# (/tmp), text summaries come back.
python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 1 > gpurun_out/tstrip_plain.log 2>&1 || exit 1
for k in exact_table_strip exact_row_carries_pipe exact_gwalk; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -f -o /tmp/rep_$k python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 1 > gpurun_out/ncu_$k.log 2>&1
python tools/ncu_top.py /tmp/rep_$k.ncu-rep 25 > gpurun_out/ncu_c3_$k.txt 2>&1
ncu -i /tmp/rep_$k.ncu-rep --page details > gpurun_out/ncu_c3_${k}_details.txt 2>&1
done
for k in exact_table_strip exact_gwalk; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -f -o /tmp/rep64_$k python tools/prof_pass.py --mode exact --radii 2 --shape 64,1024,1024 --reps 1 > gpurun_out/ncu64_$k.log 2>&1
python tools/ncu_top.py /tmp/rep64_$k.ncu-rep 25 > gpurun_out/ncu_b64_$k.txt 2>&1
ncu -i /tmp/rep64_$k.ncu-rep --page details > gpurun_out/ncu_b64_${k}_details.txt 2>&1
done
ls -la gpurun_out
