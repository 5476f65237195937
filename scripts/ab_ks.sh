# A/B of the K-split small FC (CANVAS_FC_SMALL_KS) at stage 3 / 4 shapes, then the GPU suite
mkdir -p gpurun_out/ab5
for i in 1 2; do
for v in 0 1; do
  for hw in 14 7; do
    c=$((64 * 56 / hw)); [ $hw = 7 ] && c=512
    CANVAS_FC_SMALL_KS=$v timeout 300 python scripts/kbench.py --cin $c --cout $c --hw $hw > gpurun_out/ab5/k_${hw}_v${v}_$i.txt 2>&1
    grep -E "fwd\+bwd|fc4 " gpurun_out/ab5/k_${hw}_v${v}_$i.txt | sed "s/^/$i hw$hw ks$v /"
  done
done
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/ab5/gpu_tests.log 2>&1; tail -3 gpurun_out/ab5/gpu_tests.log
timeout 600 python bench.py --no-cpu > gpurun_out/ab5/bench.log 2>&1; tail -1 gpurun_out/ab5/bench.log | cut -c1-400
