# TMEM-A forward: 8 vs 16 producer warps (unrolled k loop either way)
CANVAS_TMEMA_PW=16 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k tmem_a 2>&1 | tail -2
for i in 1 2; do
for v in 8 16; do
  CANVAS_TMEMA_PW=$v timeout 300 python scripts/kbench.py 2>&1 | grep -E "fwd\+bwd|fc9 " | sed "s/^/$i pw$v /"
done
done
