# A/B: volatile-PTX gathers on plane-major launches only (CANVAS_ASM_LOADS=planes) vs off
for i in 1 2; do
for v in 0 planes; do
  for hw in 56 28 14 7; do
    c=$((64 * 56 / hw)); [ $hw = 7 ] && c=512
    CANVAS_ASM_LOADS=$v timeout 300 python scripts/kbench.py --cin $c --cout $c --hw $hw 2>&1 | grep -E "fwd\+bwd" | sed "s/^/$i hw$hw asm$v /"
  done
done
done
