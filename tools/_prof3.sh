timeout 300 python tools/prof_kernels.py --fold-n 8 --index --reps 2 > gpurun_out/fp_plain.txt 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:fold_dense -c 1 -o gpurun_out/fold_dense_r5 python tools/prof_kernels.py --fold-n 8 --index --reps 1 > gpurun_out/ncu_fd.log 2>&1
