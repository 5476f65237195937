# TMEM-A forward at layer2 (NT = 128): 2 vs 3 operand stages (2 lets two CTAs pair on an SM), unrolled K = 1152
mkdir -p gpurun_out/ab9
CANVAS_TMEMA=1 CANVAS_TMEMA_UNROLL_MAX=1152 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "tmem_a or wide" 2>&1 | tail -2
for i in 1 2; do
for kv in "CANVAS_TMEMA=0" "CANVAS_TMEMA=1 CANVAS_TMEMA_UNROLL_MAX=1152" "CANVAS_TMEMA=1 CANVAS_TMEMA_UNROLL_MAX=1152 CANVAS_TMEMA_STAGES=3"; do
  env $kv timeout 300 python scripts/kbench.py --cin 128 --cout 128 --hw 28 2>&1 | grep -E "fc9 " | sed "s/^/$i $kv /"
done
done
