"""WKT loader checks that need no GPU.

* the device decimal parser (csrc/wkt_number.cuh), compiled as host code,
  against std::from_chars — the reference reader's number routine
  (wkt.cpp:84-95) — on a seeded fuzz corpus (tests/cpp/number_test.cpp);
* the golden WKT fixtures against the reference parse_wkt (oracle/_ref),
  which pins them: tests/golden/make_golden.py wrote them from the same
  reference.
"""
import json
import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN, ROOT


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_device_number_parser_matches_from_chars(tmp_path):
    exe = tmp_path / "number_test"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "paper_1808_09571_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "number_test.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), "400000", "7"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches=0" in r.stdout


def _cases():
    with open(os.path.join(GOLDEN, "wkt_cases.json")) as f:
        return json.load(f)


@pytest.mark.skipif(O.REF is None, reason="reference not built")
def test_golden_wkt_cases_are_the_reference_answers():
    for name, c in _cases().items():
        if c["ok"]:
            kind, coords, src = O.ref_parse_wkt(c["text"])
            assert kind == c["kind"], name
            if kind == "mesh":
                assert len(coords) == c["faces"] and O.sha_f64(coords) == c["sha"] and src == c["source"], name
        else:
            with pytest.raises(O.RefWktError) as e:
                O.ref_parse_wkt(c["text"])
            assert e.value.what == c["what"] and e.value.position == c["position"], name


def test_golden_wkt_covers_every_reference_error():
    msgs = {c["what"].rsplit(" at position", 1)[0] for c in _cases().values() if not c["ok"]}
    for m in ("expected number", "non-finite coordinate", "incomplete coordinate triple",
              "expected Z coordinate (2D input not accepted)", "interior rings are not supported",
              "polygon ring must have at least 4 points including closure",
              "polygon ring is not closed (first point != last point)",
              "TIN patch must be a triangle (4 points including closure)",
              "expected 'Z' dimension marker (2D input not accepted)", "measured coordinates are not supported",
              "empty WKT input", "trailing input after geometry", "expected '('", "expected ')'"):
        assert m in msgs, m
