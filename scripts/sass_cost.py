"""Register-read cost model of a kernel's hot loop (B200 FP64):
an FP64 instruction costs max(2, distinct 64-bit source registers not served
by the operand reuse cache) cycles (microbenchmark scripts/micro/fp64_issue.cu:
3-distinct DFMA 3.13, with a reused operand 2.05, DMUL/DADD 2.1).
usage: python scripts/sass_cost.py build/distance.o filter_kernel"""
import re, subprocess, sys

obj, name = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
body = next(f for f in funcs if name in f.split("\n", 1)[0])
ins = [(int(m.group(1), 16), m.group(2).strip()) for m in re.finditer(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", body)]
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
cost = 0.0
n3 = n3r = 0
prev_reuse = {}
other = 0
for t in best:
    t = re.sub(r"^@!?U?P\w+\s+", "", t)
    op = t.split()[0]
    args = [a.strip() for a in t[len(op):].split(",")]
    srcs = args[1:]
    reuse_now = {}
    regs = []
    for k, a in enumerate(srcs):
        m = re.match(r"[-|]*R(\d+)(\.reuse)?", a)
        if m and m.group(1) != "Z":
            r = int(m.group(1))
            if m.group(2):
                reuse_now[k] = r
            if prev_reuse.get(k) == r:
                continue  # served by the reuse cache
            regs.append(r)
    prev_reuse = reuse_now
    if op.startswith(("DFMA", "DMUL", "DADD")):
        d = len(set(regs))
        cost += max(2, d)
        if op.startswith("DFMA"):
            n3 += 1
            n3r += d >= 3
    else:
        other += 1
print(f"FP64 read-cycle estimate {cost:.0f} per warp-pair; DFMA {n3}, of which 3-distinct uncached {n3r}; other instr {other}")
