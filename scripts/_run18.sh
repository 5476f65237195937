for b in 256 32 16 8; do
timeout 300 python scripts/kbench.py --batch $b --iters 20 2>&1 | grep -E "fwd\+bwd|dgrad9 |grad7|grad1|grad0|fc9 "
done
timeout 300 python scripts/kbench.py --cin 512 --cout 512 --hw 7 --iters 10 2>&1 | grep -E "fwd\+bwd|wgrad9 "
