OSBF_GPU_EXACT=table python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 1 > gpurun_out/deep_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"col_chain_deep|exact_stencil" -s 2 -c 2 -o gpurun_out/deep2 env OSBF_GPU_EXACT=table python tools/prof_pass.py --mode exact --radii 2 --shape 1,4096,4096 --reps 1 > gpurun_out/deep_ncu.log 2>&1
echo rc=$?
