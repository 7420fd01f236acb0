"""The small-call path (direct.cu: one launch, exact composition on every
pair) and the filter/band path give the same bits on the same inputs.

Each check runs in a subprocess with TDB_DIRECT_PAIRS forcing one path: 0
(never direct) or a large limit (every one-object call and every small query
batch direct), against the golden vectors generated from the reference build
and the C oracle."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

_SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
import numpy as np
import oracle as O
import paper_1808_09571_b200 as T
from conftest import bits, GOLDEN
T.init(0)
z = np.load(GOLDEN + '/meshes.npz'); cases = {}
for k in z.files:
    name, f = k.split('/'); cases.setdefault(name, {})[f] = z[k]
for name, c in cases.items():
    if len(c['a']) * len(c['b']) > 400_000:
        continue
    r = T.mesh_mesh_distance(c['a'], c['b'])
    assert bits(r.distance) == bits(c['dist']), name
    assert (r.pair_index if r.pair_index is not None else O.U64_MAX) == int(c['pair']), name
    if r.pair_index is not None:
        assert np.array_equal(bits(np.array(r.closest_on_a)), bits(c['on_a'])), name
        assert np.array_equal(bits(np.array(r.closest_on_b)), bits(c['on_b'])), name
    h = T.mesh_mesh_intersects(c['a'], c['b'])
    assert h.hit == bool(c['hit']) and (h.pair_index if h.hit else O.U64_MAX) == int(c['hit_pair']), name
rng = np.random.default_rng(4)
for _ in range(40):
    a = rng.uniform(-1, 1, (int(rng.integers(1, 90)), 9))
    b = rng.uniform(-1, 1, (int(rng.integers(1, 90)), 9)) * rng.uniform(0.2, 1) + rng.uniform(-1.5, 1.5)
    r = T.mesh_mesh_distance(a, b)
    d, p, found, wa, wb = O.mesh_mesh_distance(a, b)
    assert bits(r.distance) == bits(d) and (r.pair_index if r.pair_index is not None else O.U64_MAX) == p
    h = T.mesh_mesh_intersects(a, b)
    hit, hp = O.mesh_mesh_intersects(a, b)
    assert h.hit == hit and (h.pair_index if h.hit else O.U64_MAX) == hp
q = dict(np.load(GOLDEN + '/queries.npz'))
m = q['ore512/mesh']
for k in range(0, 400, 7):  # small one-shot batches (1..16 queries)
    n = 1 + k % 16
    s = q['segments'][k:k + n]
    d, f = T.segments_mesh_distance(s, m)
    assert np.array_equal(bits(d), bits(q['ore512/seg_dist'][k:k + n])) and np.array_equal(f, q['ore512/seg_face'][k:k + n])
    h, hf = T.segments_mesh_intersects(s, m)
    assert np.array_equal(h, q['ore512/seg_hit'][k:k + n].astype(bool)) and np.array_equal(hf, q['ore512/seg_hit_face'][k:k + n])
    p = q['points'][k:k + n]
    d, f = T.points_mesh_distance(p, m)
    assert np.array_equal(bits(d), bits(q['ore512/pt_dist'][k:k + n])) and np.array_equal(f, q['ore512/pt_face'][k:k + n])
# near-degenerate log on both paths
sliver = np.array([[0, 0, 0, 1, 0, 0, 0.5, 1e-14, 0]], float)
far = np.array([[0, 0, 1, 1, 0, 1, 0, 1, 1.2]], float)
a = np.concatenate([T.unit_sphere(80) + 10.0, sliver])
r = T.mesh_mesh_distance(a, far)
n, ent = T.last_near_degenerate()
assert r.pair_index == 80 and n >= 1 and [0, 80] in ent.tolist()
print('DIRECT OK', T.last_stats()['kernels'])
"""


@pytest.mark.parametrize("limit", ["0", "100000000"])
def test_both_small_call_paths_bit_exact(limit):
    env = dict(os.environ, TDB_DIRECT_PAIRS=limit)
    out = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT], env=env, capture_output=True, text=True,
                         timeout=900)
    assert "DIRECT OK" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]
    kernels = int(out.stdout.split("DIRECT OK")[1].split()[0])
    assert (kernels == 1) == (limit != "0"), kernels  # the direct path is one launch
