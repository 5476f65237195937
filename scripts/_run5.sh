TAG=${1:-x}
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pinning.py tests/test_backbones.py -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/gputest.log
timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_${TAG}.log 2>&1
CANVAS_EPI_BC=0 timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_${TAG}_noepi.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_$TAG.log | cut -c1-150
for m in resnet29 mobilenet_v2; do timeout 600 python bench.py --model $m --no-cpu --steps 5 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/configs_$TAG.jsonl; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k7_bwd_wgrad9$|k3_fwd_fc9$|k5_bwd_dgrad9$|k12_bwd_grad1$|k14_bwd_grad0$" -c 5 -f -o gpurun_out/${TAG}_full python scripts/kbench.py --iters 1 > gpurun_out/ncu_full.log 2>&1
