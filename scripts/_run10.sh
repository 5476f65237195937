set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pinning.py -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/gputest.log
for i in 1 2; do
timeout 300 python scripts/kbench.py --iters 10 > gpurun_out/kb_nbr_$i.log 2>&1
CANVAS_VEC_NBR=0 timeout 300 python scripts/kbench.py --iters 10 > gpurun_out/kb_nonbr_$i.log 2>&1
done
grep -h "fwd+bwd\|fc9 \|wgrad9 \|dgrad9 " gpurun_out/kb_*.log
