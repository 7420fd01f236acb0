"""Instruction mix of a kernel's hot loop (the loop with the most FP64 ops).
usage: python scripts/sass_mix.py build/distance.o filter_kernel"""
import re, subprocess, sys
from collections import Counter

obj, name = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
body = next(f for f in funcs if name in f.split("\n", 1)[0])
ins = []
for l in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
cands = []  # innermost loops with >= 100 FP64 ops; the hot one has the most
for addr, txt in ins:
    m = re.search(r"BRA(?:\.\S+)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", txt)
    if m and int(m.group(1), 16) < addr:
        lo = int(m.group(1), 16)
        reg = [t for a, t in ins if lo <= a <= addr]
        nfp = sum(1 for t in reg if re.match(r"(@!?U?P\d+\s+)?D(FMA|MUL|ADD)", t))
        if nfp >= (int(sys.argv[3]) if len(sys.argv) > 3 else 100):
            cands.append((lo, addr, nfp, reg))
inner = [c for c in cands if not any(o is not c and c[0] <= o[0] and o[1] <= c[1] for o in cands)]
best = max(inner, key=lambda c: c[2])[3]
c = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for t in best)
fp = c["DFMA"] + c["DMUL"] + c["DADD"]
print(f"{len(best)} instructions, {fp} FP64, {len(best) - fp} other")
print(", ".join(f"{k} {v}" for k, v in c.most_common()))
