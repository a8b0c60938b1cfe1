for fam in walk stream sep; do
  OSBF_GPU_FAST=$fam python tools/prof_pass.py --radii 5,8,12,16 --shape 3,1080,1920 --reps 20 --tag c2_$fam >> gpurun_out/small2.jsonl 2>>gpurun_out/small2_err.log
  OSBF_GPU_FAST=$fam python tools/prof_pass.py --radii 5,8,16 --shape 1,1024,1024 --reps 20 --tag s1k_$fam >> gpurun_out/small2.jsonl 2>>gpurun_out/small2_err.log
  OSBF_GPU_WALK_BAND=128 OSBF_GPU_FAST=$fam python tools/prof_pass.py --radii 5,8,16 --shape 1,1024,1024 --reps 20 --tag s1k_b128_$fam >> gpurun_out/small2.jsonl 2>>gpurun_out/small2_err.log
done
