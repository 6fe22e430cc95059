timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 > gpurun_out/t_dense.log
for idx in "--index" ""; do for n in 1 8; do
echo "== idx=$idx n=$n"; timeout 300 python tools/prof_kernels.py --fold-n $n $idx --dense-permille 0 --reps 3 2>&1 | grep -E "encode|fold|Error"
done; done > gpurun_out/fold_matrix.txt 2>&1
