TAG=${1:-x}
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pinned or replication or wide" > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/gputest.log
timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_${TAG}.log 2>&1
CANVAS_EPI_PF=0 timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_${TAG}_nopf.log 2>&1
CANVAS_EPI_BC=0 timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_${TAG}_noepi.log 2>&1
grep -h "dgrad9\|grad1 \|fwd+bwd" gpurun_out/kbench_${TAG}*.log
