#!/bin/bash
# Rebuild with each -D variant and time the paper query workload (5M drills x 512-face ore).
for v in "$@"; do
  make -s lib EXTRA="$v" -B >/dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for op in distance intersects; do
    python scripts/one_query.py $op 5000000 500 2>&1 | tail -1 | python -c "
import sys,ast; l=sys.stdin.read(); d=ast.literal_eval(l[l.index('{'):]); print('$v $op: ms_total %.2f  pairs/s %.4g' % (d['ms_total'], d['pairs']/(d['ms_total']*1e-3)))"
  done
done
make -s lib -B >/dev/null 2>&1
