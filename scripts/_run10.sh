set -x
CANVAS_EPI_BC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "epilogue or pinned" > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/gputest.log
CANVAS_EPI_BC=1 timeout 300 python scripts/kbench.py --iters 10 > gpurun_out/kbench_epi_wpb2.log 2>&1
CANVAS_EPI_BC=1 CANVAS_EPI_WPB=1 timeout 300 python scripts/kbench.py --iters 10 > gpurun_out/kbench_epi_wpb1.log 2>&1
CANVAS_EPI_BC=1 CANVAS_EPI_PF=0 timeout 300 python scripts/kbench.py --iters 10 > gpurun_out/kbench_epi_wpb2_nopf.log 2>&1
timeout 300 python scripts/kbench.py --iters 10 > gpurun_out/kbench_noepi.log 2>&1
grep -h "fwd+bwd\|dgrad9 \|grad7 \|grad1 " gpurun_out/kbench_*.log
