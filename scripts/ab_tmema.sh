# A/B: FC forward with the computed operand in TMEM (fully unrolled k loop) vs the quad smem producers
mkdir -p gpurun_out/ab6
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k tmem_a 2>&1 | tail -3
for i in 1 2; do
for v in 0 1; do
  for hw in 56; do
    CANVAS_TMEMA=$v timeout 300 python scripts/kbench.py --cin 64 --cout 64 --hw $hw > gpurun_out/ab6/k_${hw}_v${v}_$i.txt 2>&1
    grep -E "fwd\+bwd|fc9 " gpurun_out/ab6/k_${hw}_v${v}_$i.txt | sed "s/^/$i hw$hw tmema$v /"
  done
done
done
