set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "image_quad or wide or pinned" > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/gputest.log
for v in "" "CANVAS_VEC_NQ=0"; do
echo "== $v"
env $v timeout 300 python scripts/kbench.py --cin 512 --cout 512 --hw 7 --iters 5 2>&1 | grep -E "fwd\+bwd|wgrad9 "
env $v timeout 300 python scripts/kbench.py --cin 256 --cout 512 --hw 14 --stride 2 --iters 5 2>&1 | grep -E "fwd\+bwd|wgrad9 "
done
