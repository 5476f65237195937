TAG=${1:-x}
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_full.log 2>&1; echo gputest=$?
tail -2 gpurun_out/gputest_full.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; tail -1 gpurun_out/bench_${TAG}.log > gpurun_out/bench_${TAG}.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.log 2>&1; tail -1 gpurun_out/bench_ref_${TAG}.log > gpurun_out/bench_ref_${TAG}.json
for m in resnet29 resnext29_2x64d mobilenet_v2 efficientnet_b0; do timeout 900 python bench.py --model $m --steps 10 --warmup 3 --ref-seconds 20 2>/dev/null | tail -1 >> gpurun_out/configs_3_5_${TAG}.jsonl; done
timeout 900 python bench.py --model vgg16 --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 >> gpurun_out/configs_3_5_${TAG}.jsonl
timeout 300 python scripts/kbench.py --iters 5 --json gpurun_out/kbench_${TAG}.json > gpurun_out/kbench_${TAG}.log 2>&1
timeout 300 python scripts/kbench.py --kernel seed7_k0 --iters 5 --json gpurun_out/kbench_k0_${TAG}.json > gpurun_out/kbench_k0_${TAG}.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-context > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k7_bwd_wgrad9$|k3_fwd_fc9$|k5_bwd_dgrad9$|k9_bwd_grad7$|k13_bwd_grad1$|k15_bwd_grad0$" -c 6 -f -o gpurun_out/${TAG}_full python scripts/kbench.py --iters 1 > gpurun_out/ncu_full.log 2>&1
bash scripts/sanitize.sh
