timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "padded or wide or image_quad or narrow or pinned or replication" > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/gputest.log
for v in "CANVAS_VEC_PAD=1" "CANVAS_VEC_PAD=0"; do
echo "== $v"
env $v timeout 300 python scripts/kbench.py --cin 512 --cout 512 --hw 7 --iters 10 2>&1 | grep -E "fwd\+bwd|fc9|wgrad9 "
env $v timeout 300 python scripts/kbench.py --kernel im2col --cin 512 --cout 512 --hw 7 --iters 10 2>&1 | grep -E "fwd\+bwd|fc|wgrad"
env $v timeout 300 python scripts/kbench.py --cin 256 --cout 512 --hw 14 --stride 2 --iters 10 2>&1 | grep -E "fwd\+bwd|fc9|wgrad9 "
done
