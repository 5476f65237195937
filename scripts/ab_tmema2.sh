# TMEM-A forward: unroll limit A/B at layer2/3 shapes (K = 1152 / 2304) + layer1, then the GPU suite
mkdir -p gpurun_out/ab7
for i in 1 2; do
for lim in 1024 2304; do
  for hw in 56 28 14; do
    c=$((64 * 56 / hw))
    CANVAS_TMEMA_UNROLL_MAX=$lim timeout 300 python scripts/kbench.py --cin $c --cout $c --hw $hw > gpurun_out/ab7/k_${hw}_l${lim}_$i.txt 2>&1
    grep -E "fwd\+bwd|fc9 " gpurun_out/ab7/k_${hw}_l${lim}_$i.txt | sed "s/^/$i hw$hw lim$lim /"
  done
done
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/ab7/gpu_tests.log 2>&1; tail -3 gpurun_out/ab7/gpu_tests.log
timeout 600 python bench.py --no-cpu > gpurun_out/ab7/bench.log 2>&1; tail -1 gpurun_out/ab7/bench.log | cut -c1-300
