# A/B: loads-first bodies with volatile PTX gathers (CANVAS_ASM_LOADS) vs compiler-scheduled __ldg
CANVAS_ASM_LOADS=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pinning.py -q -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do
for v in 0 1; do
  for hw in 56 14 7; do
    c=$((64 * 56 / hw)); [ $hw = 7 ] && c=512
    CANVAS_ASM_LOADS=$v timeout 300 python scripts/kbench.py --cin $c --cout $c --hw $hw 2>&1 | grep -E "fwd\+bwd|grad1 |grad7 |grad0 |grad4 " | sed "s/^/$i hw$hw asm$v /"
  done
done
done
