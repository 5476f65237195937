mkdir -p gpurun_out/keep2
timeout 900 python bench.py --model vgg16 --no-cpu --steps 10 --warmup 3 2>/dev/null | tail -1 > gpurun_out/keep2/vgg16.json
for i in 1 2; do timeout 900 python bench.py --no-cpu 2>/dev/null | tail -1 >> gpurun_out/keep2/bench_repeat.jsonl; done
