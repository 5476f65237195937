for v in 0 1 2; do
echo "== VEC_RT=$v"
CANVAS_VEC_RT=$v timeout 300 python scripts/kbench.py --iters 10 2>&1 | grep -E "fwd\+bwd|fc9 |wgrad9 |dgrad9 "
CANVAS_VEC_RT=$v timeout 300 python scripts/kbench.py --cin 128 --cout 128 --hw 28 --iters 10 2>&1 | grep -E "fwd\+bwd|fc9 |wgrad9 |dgrad9 "
done
