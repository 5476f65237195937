TAG=${1:-x}
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_full.log 2>&1; echo gputest=$?
tail -3 gpurun_out/gputest_full.log
timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_${TAG}.log 2>&1
CANVAS_VEC_SPLIT=0 timeout 300 python scripts/kbench.py --iters 5 > gpurun_out/kbench_${TAG}_nosplit.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_$TAG.log | cut -c1-200
bash scripts/sanitize.sh
