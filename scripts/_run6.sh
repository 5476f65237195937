TAG=${1:-x}
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pinning.py -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/gputest.log
timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_${TAG}.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_$TAG.log | cut -c1-150
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-context > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_mbv2.csv python bench.py --model mobilenet_v2 --steps 1 --warmup 3 --no-cpu --no-context > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k7_bwd_wgrad9$|k3_fwd_fc9$|k5_bwd_dgrad9$|k12_bwd_grad1$|k14_bwd_grad0$" -c 5 -f -o gpurun_out/${TAG}_full python scripts/kbench.py --iters 1 > gpurun_out/ncu_full.log 2>&1
