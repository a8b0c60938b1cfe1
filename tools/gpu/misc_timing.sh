OSBF_GPU_EXACT=table python tools/prof_pass.py --mode exact --radii 2,8 --shape 256,1024,1024 --reps 3 --tag table_c4 >> gpurun_out/misc.jsonl 2>>gpurun_out/misc_err.log
python tools/prof_pass.py --mode exact --radii 2,8 --shape 256,1024,1024 --reps 3 --tag fused_c4 >> gpurun_out/misc.jsonl 2>>gpurun_out/misc_err.log
python tools/prof_pass.py --mode fastosbf --radii 2,8 --shape 1,4096,4096 --reps 10 --tag fosbf_1 >> gpurun_out/misc.jsonl 2>>gpurun_out/misc_err.log
python tools/prof_pass.py --mode fastosbf --radii 2 --shape 256,1024,1024 --reps 3 --tag fosbf_256 >> gpurun_out/misc.jsonl 2>>gpurun_out/misc_err.log
python tools/prof_pass.py --mode box --radii 2,8 --shape 1,4096,4096 --reps 10 --tag box_1 >> gpurun_out/misc.jsonl 2>>gpurun_out/misc_err.log
python tools/prof_pass.py --mode box --radii 2 --shape 256,1024,1024 --reps 3 --tag box_256 >> gpurun_out/misc.jsonl 2>>gpurun_out/misc_err.log
python tools/prof_pass.py --mode osbf3d --radii 2 --shape 256,256,256 --reps 5 --tag osbf3d >> gpurun_out/misc.jsonl 2>>gpurun_out/misc_err.log
python tools/prof_pass.py --mode box3d --radii 2 --shape 256,256,256 --reps 5 --tag box3d >> gpurun_out/misc.jsonl 2>>gpurun_out/misc_err.log
