timeout 600 python -m pytest tests/test_gpu_codec.py tests/test_gpu_lifecycle.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/t_dense.log
timeout 300 python tools/prof_kernels.py --fold-n 8 --index --reps 2 > gpurun_out/fp_plain.txt 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:fold_list -c 1 -o gpurun_out/fold_list1 python tools/prof_kernels.py --fold-n 8 --index --reps 1 > gpurun_out/ncu_fl.log 2>&1
