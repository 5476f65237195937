set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -5 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
tail -2 gpurun_out/bench.log
