python tools/prof_pass.py --mode exact --radii 2 --shape 64,1024,1024 --reps 1 > gpurun_out/strip_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:exact_strip -s 2 -c 1 -o gpurun_out/strip2 python tools/prof_pass.py --mode exact --radii 2 --shape 64,1024,1024 --reps 1 > gpurun_out/strip_ncu.log 2>&1
echo rc=$?
