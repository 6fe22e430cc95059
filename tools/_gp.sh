timeout 900 python tools/grad_bench.py --reps 1 > gpurun_out/gb_plain.json 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:adam_replay -c 1 -o gpurun_out/grad_r3 python tools/grad_bench.py --reps 1 > gpurun_out/ncu_grad.log 2>&1
