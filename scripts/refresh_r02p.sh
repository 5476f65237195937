# Final round-2 refresh (r02p): GPU tests, bench (+ reference arm), configs 3/5, layer1/layer4
# kbench, config 1, launch list, ncu --set full of the layer1 Canvas kernels, compute-sanitizer
set -x
K=gpurun_out/keep2
mkdir -p $K
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $K/gpu_tests.log 2>&1; tail -3 $K/gpu_tests.log
timeout 900 python bench.py > $K/bench.log 2>&1; tail -1 $K/bench.log > $K/bench.json
timeout 600 python bench.py --impl reference > $K/bench_ref.log 2>&1; tail -1 $K/bench_ref.log > $K/bench_ref.json
for m in resnet29 resnext29_2x64d mobilenet_v2 efficientnet_b0; do timeout 900 python bench.py --model $m --steps 10 --warmup 3 2>/dev/null | tail -1 >> $K/configs_3_5.jsonl; done
timeout 900 python bench.py --model vgg16 --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 >> $K/configs_3_5.jsonl
timeout 300 python scripts/kbench.py --json $K/kbench_layer1.json > $K/kbench_layer1.txt 2>&1
timeout 300 python scripts/kbench.py --cin 512 --cout 512 --hw 7 --json $K/kbench_layer4.json > $K/kbench_layer4.txt 2>&1
for k in seed7_k1 seed7_k0 im2col; do timeout 300 python scripts/kbench.py --kernel $k --batch 8 --iters 20 --json $K/config1_$k.json > $K/config1_$k.txt 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $K/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-context > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k7_bwd_wgrad9$|k3_fwd_fc9$|k5_bwd_dgrad9$|k9_bwd_grad7$|k13_bwd_grad1$|k15_bwd_grad0$" -c 6 -f -o $K/full python scripts/kbench.py --iters 1 > $K/ncu_full.log 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 600 compute-sanitizer --tool $t --print-limit 20 --error-exitcode 9 python scripts/sanitize.py > $K/sanitizer_$t.txt 2>&1
  echo "$t exit=$?" | tee -a $K/sanitizer_summary.txt
  tail -3 $K/sanitizer_$t.txt >> $K/sanitizer_summary.txt
done
ls -la $K
