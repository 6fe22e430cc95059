timeout 900 python tools/grad_bench.py --reps 1 > gpurun_out/gb_plain.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/grad_launches.csv python tools/grad_bench.py --reps 1 > gpurun_out/ncu_gl.log 2>&1
