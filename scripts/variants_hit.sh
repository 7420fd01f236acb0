#!/bin/bash
# Rebuild with each -D variant and time one C3 intersects call (131,072 rows).
for v in "$@"; do
  make -s lib EXTRA="$v" -B >/dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"; python scripts/one_call.py intersects 131072 2>&1 | tail -1 | python -c "
import sys,ast; l=sys.stdin.read(); d=ast.literal_eval(l[l.index('{'):]); print('pairs/s %.4g  ms %.1f' % (d['pairs']/(d['ms_filter']*1e-3), d['ms_filter']))"
done
make -s lib -B >/dev/null 2>&1
