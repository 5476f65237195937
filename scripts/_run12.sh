for v in 1 0; do echo "== PAD=$v"; CANVAS_VEC_PAD=$v timeout 600 python scripts/_dbg_pad.py 2>&1 | tail -25; done
