# A/B of CANVAS_LOADS_FIRST (gathers hoisted above the arithmetic in pointwise bodies)
mkdir -p gpurun_out/ab4
for i in 1 2; do
for v in 0 1; do
  for hw in 56 14 7; do
    c=$((64 * 56 / hw)); [ $hw = 7 ] && c=512
    CANVAS_LOADS_FIRST=$v timeout 300 python scripts/kbench.py --cin $c --cout $c --hw $hw > gpurun_out/ab4/k_${hw}_v${v}_$i.txt 2>&1
    grep -E "fwd\+bwd|grad|softmax|bcast" gpurun_out/ab4/k_${hw}_v${v}_$i.txt | sed "s/^/$i hw$hw lf$v /"
  done
done
done
