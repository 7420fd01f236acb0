#!/bin/bash
# Rebuild distance.o with each -D switch set and time the default bench
# (C2, 3 timed steps after 2 warm-up steps, no CPU leg, no e2e leg).
# usage: scripts/variants_bench.sh "-DX=1" "-DX=2" ...
for v in "$@"; do
  touch paper_1808_09571_b200/csrc/distance.cu
  make -s lib EXTRA="$v" >/dev/null 2>&1 || { echo "build failed: $v"; continue; }
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('%-60s %.4g pairs/s  %.1f ms/step' % ('$v', d['value'], d['ms_per_step']))"
done
touch paper_1808_09571_b200/csrc/distance.cu
make -s lib >/dev/null 2>&1
