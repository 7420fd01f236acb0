"""GPU parity: the device WKT loader (csrc/wkt.cu) against the reference
parse_wkt (wkt.cpp:188).

Accepted literals must give the reference's triangles bit for bit (sha of
the face array, from tests/golden/wkt_cases.json, written by the reference);
rejected literals must raise the reference's WktParseError message at the
same byte position. At full size: the reference serializer's canonical text
of the 1.31M-face ore body parses back to the generator's exact bits
(serialize/parse round trip, wkt.hpp:38-40).
"""
import json
import os
import time

import numpy as np
import pytest

import oracle as O
import paper_1808_09571_b200 as T
from conftest import GOLDEN, bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def device():
    T.init(0)
    yield


@pytest.fixture(scope="module")
def cases():
    with open(os.path.join(GOLDEN, "wkt_cases.json")) as f:
        return json.load(f)


def test_golden_literals(cases):
    for name, c in cases.items():
        if c["ok"] and c["kind"] == "mesh":
            m = T.mesh_from_wkt(c["text"])
            got = m.download()
            assert len(got) == c["faces"] and O.sha_f64(got) == c["sha"], name
        elif c["ok"]:  # POINT / LINESTRING: valid WKT, not a mesh
            with pytest.raises(T.WktParseError, match="not a mesh"):
                T.mesh_from_wkt(c["text"])
        else:
            with pytest.raises(T.WktParseError) as e:
                T.mesh_from_wkt(c["text"])
            assert (e.value.what, e.value.position) == (c["what"], c["position"]), name


def test_table_of_literals_and_first_bad_literal(cases):
    good = [c["text"] for c in cases.values() if c["ok"] and c["kind"] == "mesh"]
    want = [T.mesh_from_wkt(t).download() for t in good]
    tab = T.table_from_wkt(good * 3)
    got = tab.download()
    assert np.array_equal(bits(got), bits(np.concatenate(want * 3)))
    assert tab.info()["objects"] == 3 * len(good)
    bad = [(n, c) for n, c in cases.items() if not c["ok"] and c["text"].strip()]
    for name, c in bad[:12]:
        lits = good + [c["text"]] + good
        with pytest.raises(T.WktParseError) as e:
            T.table_from_wkt(lits)
        assert e.value.literal == len(good), name
        assert (e.value.what, e.value.position) == (c["what"], c["position"]), name


def test_loaded_mesh_runs_the_operators(cases):
    s = T.unit_sphere(1000)
    m = T.mesh_from_wkt(cases["sphere_canonical"]["text"])
    b = T.translate(s, 2.5)
    r1 = T.mesh_mesh_distance(m, b)
    r2 = T.mesh_mesh_distance(s, b)
    assert bits(r1.distance) == bits(r2.distance) and r1.pair_index == r2.pair_index


@pytest.mark.skipif(O.REF is None, reason="reference serializer (oracle/_ref) not built")
def test_full_size_ore_round_trip():
    ore = T.ore_body(1_000_000)  # 1,310,720 faces
    text = O.ref_serialize_mesh(ore, as_bytes=True)  # the reference's canonical TIN Z text
    T.mesh_from_wkt(text[:100_000].rsplit(b"((", 1)[0].rstrip(b", ") + b")")  # warm-up
    t = time.perf_counter()
    m = T.mesh_from_wkt(text)
    dt = time.perf_counter() - t
    got = m.download()
    assert np.array_equal(bits(got), bits(ore))
    print(f"\nWKT load {len(text) / 1e6:.0f} MB -> {len(got)} faces in {dt * 1e3:.1f} ms "
          f"({len(text) / dt / 1e9:.2f} GB/s)")
