#!/bin/bash
# Like variants.sh, but rebuilds only distance.o (for -D switches that only
# distance.cu reads: TDB_FILTER_MINB, TDB_UV / TDB_UF / TDB_UE).
# usage: scripts/variants_dist.sh ROWS "-DX=1" "-DX=2" ...
rows=$1; shift
for v in "$@"; do
  touch paper_1808_09571_b200/csrc/distance.cu
  make -s lib EXTRA="$v" >/dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"; python scripts/one_call.py distance $rows 2>&1 | tail -1 | python -c "
import sys,ast; l=sys.stdin.read(); d=ast.literal_eval(l[l.index('{'):]); print('pairs/s %.4g  ms_filter %.1f' % (d['pairs']/(d['ms_filter']*1e-3), d['ms_filter']))"
done
touch paper_1808_09571_b200/csrc/distance.cu
make -s lib >/dev/null 2>&1
