set -x
for i in 1 2; do
timeout 300 python scripts/kbench.py --iters 10 > gpurun_out/kbench_nofmad_$i.log 2>&1
CANVAS_FMAD=1 timeout 300 python scripts/kbench.py --iters 10 > gpurun_out/kbench_fmad_$i.log 2>&1
done
grep -h "fwd+bwd\|fc9 \|wgrad9 \|grad1 " gpurun_out/kbench_*fmad_*.log
