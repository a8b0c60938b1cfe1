R=${1:-20}
python tools/prof_pass.py --radii $R --shape 1,16384,16384 --reps 1 > gpurun_out/ncu_vwalk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fast_vwalk -s 3 -c 1 -o gpurun_out/vwalk_r$R \
    python tools/prof_pass.py --radii $R --shape 1,16384,16384 --reps 1 > gpurun_out/ncu_vwalk.log 2>&1
echo rc=$?
