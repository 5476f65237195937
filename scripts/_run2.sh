# usage: bash scripts/_run2.sh TAG [tests]
TAG=${1:-x}
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
if [ "$2" != "notests" ]; then
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pinning.py tests/test_dense_conv.py -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/gputest.log
fi
timeout 600 python bench.py --no-cpu > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_$TAG.log
timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k7_bwd_wgrad9$|k3_fwd_fc9$|k5_bwd_dgrad9$|k9_bwd_grad7$|k13_bwd_grad1$|k15_bwd_grad0$" -c 6 -f -o gpurun_out/${TAG}_full python scripts/kbench.py --iters 1 > gpurun_out/ncu_full.log 2>&1
