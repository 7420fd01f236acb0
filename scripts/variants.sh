#!/bin/bash
# Rebuild the library with each -D variant and time one C2 distance call.
# usage: scripts/variants.sh ROWS "-DX=1" "-DX=2" ...
rows=$1; shift
for v in "$@"; do
  make -s lib EXTRA="$v" -B >/dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"; python scripts/one_call.py distance $rows 2>&1 | tail -1 | python -c "
import sys,ast; l=sys.stdin.read(); d=ast.literal_eval(l[l.index('{'):]); print('pairs/s %.4g  ms_filter %.1f' % (d['pairs']/(d['ms_filter']*1e-3), d['ms_filter']))"
done
make -s lib -B >/dev/null 2>&1
