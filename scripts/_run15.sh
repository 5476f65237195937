timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1; echo gpu_all=$?
tail -3 gpurun_out/gpu_all.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -c 1500 gpurun_out/bench.json
