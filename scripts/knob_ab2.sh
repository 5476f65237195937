# A/B of wgrad knobs, alternated on one box (results in gpurun_out/knob_ab2.txt)
mkdir -p gpurun_out
for rep in 1 2; do
for kv in BASE=1 CANVAS_WGRAD_TCHUNK=16384 CANVAS_WGRAD_JG=1 CANVAS_WGRAD_JG=3 CANVAS_PLANES_MIN_S=256; do
  env $kv timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu --no-context 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$kv', d['value'], d['e2e']['value'], d['ms_per_step'])" >> gpurun_out/knob_ab2.txt 2>&1 || echo "$kv failed" >> gpurun_out/knob_ab2.txt
done; done
cat gpurun_out/knob_ab2.txt
