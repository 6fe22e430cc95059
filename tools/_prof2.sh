timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2 > gpurun_out/t_all.log
timeout 600 python bench.py --no-e2e --cpu-baseline 0 --restore-chain 0 --steps 2 --warmup 3 > gpurun_out/p_plain.json 2>gpurun_out/p_plain.err && \
timeout 2000 ncu --set full --import-source on --clock-control none -k regex:"encode_mask|encode_emit|fold_kernel" -c 3 -o gpurun_out/full_r5 python bench.py --no-e2e --cpu-baseline 0 --restore-chain 0 --steps 2 --warmup 3 > gpurun_out/p_ncu2.log 2>&1
