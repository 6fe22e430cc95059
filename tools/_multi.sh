timeout 600 python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -2 > gpurun_out/t_multi.log
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
done
