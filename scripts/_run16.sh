for v in 1; do
echo "== SIB=$v"
CANVAS_GRAD_SIBLINGS=$v timeout 300 python scripts/kbench.py --iters 10 2>&1 | grep -E "fwd\+bwd|grad"
done
