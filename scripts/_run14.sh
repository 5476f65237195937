for k in seed7_k1 im2col involution; do
for v in "CANVAS_VEC_PAD=1" "CANVAS_VEC_PAD=0"; do
echo "== $k $v"
env $v timeout 300 python scripts/kbench.py --kernel $k --cin 512 --cout 512 --hw 7 --iters 10 2>&1 | grep -E "fwd\+bwd|wgrad"
env $v timeout 300 python scripts/kbench.py --kernel $k --cin 256 --cout 512 --hw 14 --stride 2 --iters 10 2>&1 | grep -E "fwd\+bwd|wgrad"
done; done
for f in 3 11 17 40 77; do
python - $f <<'PY' > /tmp/k$f.cir
import sys
t=open("tests/golden/sampler_10_7_256.cir").read().split("canvas-ir v1\n")[1:]
sys.stdout.write("canvas-ir v1\n"+t[int(sys.argv[1])])
PY
for v in "CANVAS_VEC_PAD=1" "CANVAS_VEC_PAD=0"; do
echo "== sweep#$f $v"
env $v timeout 300 python scripts/kbench.py --kernel /tmp/k$f.cir --cin 512 --cout 512 --hw 7 --iters 10 2>&1 | grep -E "fwd\+bwd|tc wgrad"
done; done
