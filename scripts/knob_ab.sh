# A/B of candidate knob defaults, alternated on one box (results in gpurun_out/knob_ab.txt)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for rep in 1 2; do
for kv in BASE=1 CANVAS_WGRAD_TCHUNK=8192 "CANVAS_WGRAD_TCHUNK=8192 CANVAS_TC_PW=16"; do
  env $kv timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu --no-context 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$kv', d['value'], d['e2e']['value'], d['ms_per_step'])" >> gpurun_out/knob_ab.txt 2>&1 || echo "$kv failed" >> gpurun_out/knob_ab.txt
done; done
cat gpurun_out/knob_ab.txt
