# Round-end refresh: GPU tests, bench (+ reference arm), launch list and ncu --set full of the layer1 Canvas kernels
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_final.log 2>&1; tail -3 gpurun_out/gpu_tests_final.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; tail -1 gpurun_out/bench_final.log > gpurun_out/bench_final.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01f.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-context > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k7_bwd_wgrad9$|k3_fwd_fc9$|k5_bwd_dgrad9$|k9_bwd_grad7$|k13_bwd_grad1$|k15_bwd_grad0$" -c 6 -f -o gpurun_out/r01f_full python scripts/kbench.py --iters 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
