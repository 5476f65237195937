TAG=${1:-x}
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pinning.py tests/test_dense_conv.py -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/gputest.log
timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_${TAG}.log 2>&1
CANVAS_PLANES_GUARDED=1 timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_${TAG}_pg.log 2>&1
CANVAS_PLANES_GUARDED=1 CANVAS_VEC_SHIFTED=1 timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_${TAG}_pgv.log 2>&1
CANVAS_VEC_SHIFTED=1 timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_${TAG}_v.log 2>&1
timeout 300 python scripts/kbench.py --kernel seed7_k0 --batch 8 --iters 20 > gpurun_out/kbench_${TAG}_k0b8.log 2>&1
CANVAS_GRAD_INLINE=0 CANVAS_FOLD_INLINE=0 timeout 300 python scripts/kbench.py --kernel seed7_k0 --batch 8 --iters 20 > gpurun_out/kbench_${TAG}_k0b8_noinl.log 2>&1
timeout 300 python scripts/kbench.py --kernel seed7_k0 --iters 5 > gpurun_out/kbench_${TAG}_k0.log 2>&1
CANVAS_GRAD_INLINE=0 CANVAS_FOLD_INLINE=0 timeout 300 python scripts/kbench.py --kernel seed7_k0 --iters 5 > gpurun_out/kbench_${TAG}_k0_noinl.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_$TAG.log | cut -c1-120
for m in mobilenet_v2 vgg16; do timeout 900 python bench.py --model $m --no-cpu --steps 5 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/configs_$TAG.jsonl; done
