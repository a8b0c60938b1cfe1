python tools/prof_pass.py --mode osbf3d --radii 2 --shape 256,256,256 --reps 1 > gpurun_out/p3d_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p3d_launches.csv python tools/prof_pass.py --mode osbf3d --radii 2 --shape 256,256,256 --reps 1 > gpurun_out/p3d_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:filter3d -s 2 -c 1 -o gpurun_out/f3d python tools/prof_pass.py --mode osbf3d --radii 2 --shape 256,256,256 --reps 1 > gpurun_out/p3d_ncu2.log 2>&1
echo rc=$?
