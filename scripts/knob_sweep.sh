# One bench line per lowering knob setting (scripts/knob_sweep.sh; results in gpurun_out/knobs.txt)
mkdir -p gpurun_out
for kv in BASE=1 CANVAS_PW_VEC=2 CANVAS_TC_PW=16 CANVAS_WGRAD_TCHUNK=2048 CANVAS_WGRAD_TCHUNK=8192 CANVAS_PLANES_CTAS=4736 CANVAS_TC_NTMAX=128 CANVAS_WGRAD_PW=8 BASE=2; do
  env $kv timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-context 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$kv', d['value'], d['e2e']['value'], d['ms_per_step'])" >> gpurun_out/knobs.txt 2>&1 || echo "$kv failed" >> gpurun_out/knobs.txt
done
cat gpurun_out/knobs.txt
