for i in 1 2; do timeout 900 python bench.py --no-cpu --no-context 2>/dev/null | tail -1 >> gpurun_out/r21_bench.jsonl; done
for v in "CANVAS_PIX_PW=0" "CANVAS_PIX_PW=16" "CANVAS_TC_PAIR=0"; do
echo "== $v"
env $v timeout 300 python scripts/kbench.py --iters 10 2>&1 | grep -E "fwd\+bwd|fc9 "
env $v timeout 300 python scripts/kbench.py --cin 128 --cout 128 --hw 28 --iters 10 2>&1 | grep -E "fwd\+bwd|fc9 "
env $v timeout 300 python scripts/kbench.py --cin 256 --cout 256 --hw 14 --iters 10 2>&1 | grep -E "fwd\+bwd|fc9 "
done
