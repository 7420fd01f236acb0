"""The per-pair operation counts bench.py reports (fp32_instr_per_pair,
fp64_instr_per_pair) against the SASS of the built kernels: the hot loop of
edge32_kernel (packed FP32 edge/edge candidates) and of vertex_kernel. CPU
only (cuobjdump on build/distance.o); skipped when the object is absent."""
import os
import re
import shutil
import subprocess
from collections import Counter

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "build", "distance.o")


def _hot_loop(name, marker):
    sass = subprocess.run(["cuobjdump", "-sass", OBJ], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)
    body = next(f for f in funcs if name in f.split("\n", 1)[0])
    ins = [(int(m.group(1), 16), m.group(2).strip())
           for m in re.finditer(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", body)]
    loops = []
    for addr, txt in ins:
        m = re.search(r"BRA(?:\.\S+)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", txt)
        if m and int(m.group(1), 16) < addr:
            lo = int(m.group(1), 16)
            ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for a, t in ins if lo <= a <= addr)
            if ops.get(marker, 0):
                loops.append((lo, addr, ops))
    # innermost loop carrying the marker
    inner = [l for l in loops if not any(o is not l and l[0] <= o[0] and o[1] <= l[1] for o in loops)]
    return max(inner, key=lambda l: l[2][marker])[2]


needs_obj = pytest.mark.skipif(not (os.path.exists(OBJ) and shutil.which("cuobjdump")),
                               reason="build/distance.o or cuobjdump absent")


@needs_obj
def test_edge32_ops_per_pair_match_bench():
    import bench
    ops = _hot_loop("edge32_kernel", "FFMA2")
    pairs = ops["FMNMX"]  # one running-minimum update per edge pair
    fp32 = 2 * ops["FFMA2"] + 2 * ops["FMUL2"] + 2 * ops["FADD2"] + ops["FMUL.SAT"] + ops["FMNMX"]
    flops = 4 * ops["FFMA2"] + 2 * ops["FMUL2"] + 2 * ops["FADD2"] + ops["FMUL.SAT"]
    assert ops["MUFU.RCP"] == pairs
    assert fp32 / pairs == bench.FILTER_EDGE_PAIR32[0], (dict(ops), fp32 / pairs)
    assert flops / pairs == bench.FILTER_EDGE_PAIR32[1], (dict(ops), flops / pairs)


@needs_obj
def test_vertex_kernel_ops_per_pair_match_bench():
    import bench
    ops = _hot_loop("vertex_kernel", "DFMA")
    pairs = ops["VIMNMX"]  # one running-minimum update per (A vertex, B face)
    fp64 = ops["DFMA"] + ops["DMUL"] + ops["DADD"]
    flops = 2 * ops["DFMA"] + ops["DMUL"] + ops["DADD"]
    assert fp64 / pairs == bench.FILTER_VERT_PAIR[0], (dict(ops), fp64 / pairs)
    assert flops / pairs == bench.FILTER_VERT_PAIR[1], (dict(ops), flops / pairs)
