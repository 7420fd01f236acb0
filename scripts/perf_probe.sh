#!/bin/bash
# quick perf probe: distance C2 rows and intersects C3 rows (resident meshes)
python scripts/one_call.py distance ${1:-16384} 2>&1 | tail -1 | python -c "
import sys,ast; l=sys.stdin.read(); d=ast.literal_eval(l[l.index('{'):]); print('distance   pairs/s %.4g  ms_filter %.1f  cand %d' % (d['pairs']/(d['ms_filter']*1e-3), d['ms_filter'], d['candidates']))"
python scripts/one_call.py intersects ${2:-131072} 2>&1 | tail -1 | python -c "
import sys,ast; l=sys.stdin.read(); d=ast.literal_eval(l[l.index('{'):]); print('intersects pairs/s %.4g  ms %.1f  exact %d' % (d['pairs']/(d['ms_filter']*1e-3), d['ms_filter'], d['exact_pairs']))"
