set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "narrow or replication or pinned" > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/gputest.log
timeout 300 python scripts/kbench.py --cin 24 --cout 144 --hw 56 --k 1 --iters 5 > gpurun_out/kb_mb1.log 2>&1
timeout 300 python scripts/kbench.py --cin 144 --cout 24 --hw 56 --k 1 --iters 5 > gpurun_out/kb_mb2.log 2>&1
grep -h "fwd+bwd\|wgrad9 \|fc9 " gpurun_out/kb_mb*.log
for m in mobilenet_v2 efficientnet_b0 resnet29; do timeout 900 python bench.py --model $m --no-cpu --steps 5 --warmup 3 2>/dev/null | tail -1 | cut -c1-200; done
