set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pinned or wide or narrow" > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/gputest.log
for v in "CANVAS_TMEMA_PW=16" "CANVAS_TMEMA_PW=8" "CANVAS_TMEMA=0"; do
echo "== $v"
env $v timeout 300 python scripts/kbench.py --iters 10 2>&1 | grep -E "fwd\+bwd|fc9 "
env $v timeout 300 python scripts/kbench.py --cin 128 --cout 128 --hw 28 --iters 5 2>&1 | grep -E "fc9 "
done
