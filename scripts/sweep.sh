#!/bin/bash
# All bench configurations back to back (one B200), one summary line each;
# the raw JSON lines go to gpurun_out/sweep.jsonl. Used for DESIGN.md section 6.
mkdir -p gpurun_out
: > gpurun_out/sweep.jsonl
for c in "--config c1" "--config c2" "--config c3 --steps 4" "--config c3s --steps 2" "--config c4 --steps 4 --e2e-steps 2" \
         "--config c5 --steps 2 --e2e-steps 1" "--config paper --steps 8" "--config paper --op intersects --steps 8" \
         "--config c2 --mode cull --steps 4 --no-cpu"; do
  timeout 900 python bench.py $c 2>/dev/null | tail -1 | tee -a gpurun_out/sweep.jsonl | python -c "
import sys, json
d = json.loads(sys.stdin.read()); r = d['roofline']; cb = d.get('cpu_baseline') or {}
print('%-45s value %.3g e2e %.3g ms/step %.2f frac %.3g cpu %s' % ('$c', d['value'], d['e2e']['value'], d['ms_per_step'], r['frac'], cb.get('value')))"
done
