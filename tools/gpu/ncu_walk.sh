# ncu --set full of one fast_walk_step launch on the 32768^2 plane (r = $1)
R=${1:-4}
export OSBF_GPU_FAST=walk
python tools/prof_pass.py --radii $R --shape 1,32768,32768 --reps 1 > gpurun_out/ncu_walk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fast_walk -s 3 -c 1 -o gpurun_out/walk_r$R \
    python tools/prof_pass.py --radii $R --shape 1,32768,32768 --reps 1 > gpurun_out/ncu_walk.log 2>&1
echo rc=$?
