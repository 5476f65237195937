# A/B of the per-pixel small FC forward: quads (pointwise4) vs one pixel per thread
mkdir -p gpurun_out/ab3
for i in 1 2; do
for kv in "CANVAS_FC_SMALL_VEC_FILL=2048" "CANVAS_FC_SMALL_VEC_FILL=256" "CANVAS_FC_SMALL_VEC_FILL=256 CANVAS_FC_SMALL_UNROLL=16"; do
  for hw in 56 28 14; do
    c=$((64 * 56 / hw))
    env $kv timeout 300 python scripts/kbench.py --cin $c --cout $c --hw $hw 2>&1 | grep -E "fc4 " | sed "s/^/$i hw$hw $kv /"
  done
done
done
