# Round-2 refresh (r02o): GPU tests, bench (+ reference arm), configs 3/5, launch list, ncu --set full of the layer1 Canvas kernels
set -x
mkdir -p gpurun_out/keep
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/keep/gpu_tests.log 2>&1; tail -3 gpurun_out/keep/gpu_tests.log
timeout 900 python bench.py > gpurun_out/keep/bench.log 2>&1; tail -1 gpurun_out/keep/bench.log > gpurun_out/keep/bench.json
timeout 600 python bench.py --impl reference > gpurun_out/keep/bench_ref.log 2>&1; tail -1 gpurun_out/keep/bench_ref.log > gpurun_out/keep/bench_ref.json
for m in resnet29 resnext29_2x64d mobilenet_v2 efficientnet_b0 vgg16; do timeout 900 python bench.py --model $m --steps 10 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/keep/configs_3_5.jsonl; done
timeout 300 python scripts/kbench.py --json gpurun_out/keep/kbench_layer1.json > gpurun_out/keep/kbench_layer1.txt 2>&1
timeout 300 python scripts/kbench.py --cin 512 --cout 512 --hw 7 --json gpurun_out/keep/kbench_layer4.json > gpurun_out/keep/kbench_layer4.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/keep/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-context > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k7_bwd_wgrad9$|k3_fwd_fc9$|k5_bwd_dgrad9$|k9_bwd_grad7$|k13_bwd_grad1$|k15_bwd_grad0$" -c 6 -f -o gpurun_out/keep/full python scripts/kbench.py --iters 1 > gpurun_out/keep/ncu_full.log 2>&1
ls -la gpurun_out/keep
