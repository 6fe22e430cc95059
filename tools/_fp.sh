timeout 600 python -m pytest tests/test_gpu_codec.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/t_dense.log
for idx in "" "--index"; do for n in 1 8; do for p in 0; do
echo "== idx=$idx n=$n p=$p"; timeout 300 python tools/prof_kernels.py --fold-n $n $idx --dense-permille $p --reps 3 2>&1 | grep -E "fold|Error"
done; done; done > gpurun_out/fold_matrix.txt 2>&1
