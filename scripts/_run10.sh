set -x
python scripts/case20_5.py 5
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pinning.py -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/gputest.log
timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_rn.log 2>&1
grep -h "fwd+bwd\|softmax" gpurun_out/kbench_rn.log
timeout 300 python scripts/kbench.py --cin 512 --cout 512 --hw 7 --iters 5 > gpurun_out/kbench_rn7.log 2>&1
CANVAS_FMAD=0 timeout 300 python scripts/kbench.py --cin 512 --cout 512 --hw 7 --iters 5 > gpurun_out/kbench_nofmad7.log 2>&1
grep -h "fwd+bwd\|softmax" gpurun_out/kbench_rn7.log gpurun_out/kbench_nofmad7.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_rn.log 2>&1
tail -1 gpurun_out/bench_rn.log | cut -c1-130
