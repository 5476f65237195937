# A/B of the per-pixel small FC forward variants on one box
mkdir -p gpurun_out/ab2
for i in 1 2; do
for kv in "CANVAS_FC_SMALL_UNROLL=0" "CANVAS_FC_SMALL_W4=1" "CANVAS_FC_SMALL_UNROLL=8" "CANVAS_FC_SMALL_UNROLL=16" "CANVAS_FC_SMALL_UNROLL=64"; do
  for hw in 56 28; do
    c=$((64 * 56 / hw))
    env $kv timeout 300 python scripts/kbench.py --cin $c --cout $c --hw $hw 2>&1 | grep -E "fc4 " | sed "s/^/$i hw$hw $kv /"
  done
done
done
