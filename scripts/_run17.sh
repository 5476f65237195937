timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pinned or wide or padded" > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/gputest.log
for k in seed7_k1 im2col involution; do
for v in 1 0; do
echo "== $k KEYS=$v"
CANVAS_ROW_KEYS=$v timeout 300 python scripts/kbench.py --kernel $k --iters 10 2>&1 | grep -E "fwd\+bwd|tc wgrad"
CANVAS_ROW_KEYS=$v timeout 300 python scripts/kbench.py --kernel $k --cin 128 --cout 128 --hw 28 --iters 10 2>&1 | grep -E "fwd\+bwd|tc wgrad"
done; done
