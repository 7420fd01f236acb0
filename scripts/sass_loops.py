"""Per-loop instruction mix of a kernel (innermost loops with FP64 work):
instructions, DFMA / DMUL / DADD, executed FP64 flops, and the register-read
cost model of scripts/sass_cost.py. For filter_kernel<false> (FULL mode) the
loops are the vertex and face candidate loops; for edge_kernel the edge/edge
loop (unrolled: divide by its unroll factor). bench.py's FILTER_LOOP_*
constants come from here.
usage: python scripts/sass_loops.py build/distance.o filter_kernelILb0   (name: regex)"""
import re, subprocess, sys
from collections import Counter

obj, name = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
body = next(f for f in funcs if re.search(name, f.split("\n", 1)[0]))
ins = [(int(m.group(1), 16), m.group(2).strip()) for m in re.finditer(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", body)]
loops = []
for addr, txt in ins:
    m = re.search(r"BRA(?:\.\S+)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", txt)
    if m and int(m.group(1), 16) < addr:
        lo = int(m.group(1), 16)
        reg = [t for a, t in ins if lo <= a <= addr]
        if sum(1 for t in reg if re.match(r"(@!?U?P\d+\s+)?D(FMA|MUL|ADD)", t)) >= 5:
            loops.append((lo, addr, reg))
inner = [c for c in loops if not any(o is not c and c[0] <= o[0] and o[1] <= c[1] for o in loops)]
for lo, hi, reg in sorted(inner):
    c = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for t in reg)
    cost, prev = 0.0, {}
    for t in reg:
        t = re.sub(r"^@!?U?P\w+\s+", "", t)
        op = t.split()[0]
        srcs = [a.strip() for a in t[len(op):].split(",")][1:]
        now, regs = {}, []
        for k, a in enumerate(srcs):
            m = re.match(r"[-|]*R(\d+)(\.reuse)?", a)
            if m:
                r = int(m.group(1))
                if m.group(2):
                    now[k] = r
                if prev.get(k) != r:
                    regs.append(r)
        prev = now
        if op.startswith(("DFMA", "DMUL", "DADD")):
            cost += max(2, len(set(regs)))
    fp = c["DFMA"] + c["DMUL"] + c["DADD"]
    print(f"loop {lo:#x}-{hi:#x}: {len(reg)} instr, FP64 {fp} (DFMA {c['DFMA']}, DMUL {c['DMUL']}, DADD {c['DADD']}), "
          f"flops {2 * c['DFMA'] + c['DMUL'] + c['DADD']}, read-cycle estimate {cost:.0f}")
