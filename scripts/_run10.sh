set -x
CANVAS_VEC_RT=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pinning.py -x -q -p no:cacheprovider -k "pinned or replication or wide or narrow or sweep256 or bench_layer" > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/gputest.log
for i in 1 2; do
CANVAS_VEC_RT=2 timeout 300 python scripts/kbench.py --iters 10 > gpurun_out/kbench_rt2_$i.log 2>&1
timeout 300 python scripts/kbench.py --iters 10 > gpurun_out/kbench_rt0_$i.log 2>&1
done
grep -h "fwd+bwd\|fc9 \|wgrad9 " gpurun_out/kbench_rt*.log
