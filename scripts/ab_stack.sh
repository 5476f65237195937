# A/B: stacked-N wgrad MMA (hi.hi + hi.lo as one N = 2 NT MMA) vs 3 MMAs, then the GPU suite
mkdir -p gpurun_out/ab8
CANVAS_WGRAD_STACK=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pinning.py -q -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do
for v in 0 1; do
  for hw in 56 28; do
    c=$((64 * 56 / hw))
    CANVAS_WGRAD_STACK=$v timeout 300 python scripts/kbench.py --cin $c --cout $c --hw $hw > gpurun_out/ab8/k_${hw}_v${v}_$i.txt 2>&1
    grep -E "fwd\+bwd|wgrad9 " gpurun_out/ab8/k_${hw}_v${v}_$i.txt | sed "s/^/$i hw$hw stack$v /"
  done
done
done
