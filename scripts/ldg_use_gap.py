"""Flag global loads whose destination register is read within N instructions
(the consumer waits on the load's full latency).
Usage: python scripts/ldg_use_gap.py lib.so FUNC_REGEX [N]"""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
pat = re.compile(sys.argv[2])
N = int(sys.argv[3]) if len(sys.argv) > 3 else 6
cur, ins = None, []
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and cur and pat.search(cur):
        ins.append((cur, m.group(1), m.group(2).strip()))
for i, (fn, addr, txt) in enumerate(ins):
    m = re.search(r"LDG\S*\s+(R\d+),", txt)
    if not m:
        continue
    r = m.group(1)
    for j in range(i + 1, min(i + 1 + N, len(ins))):
        if ins[j][0] != fn:
            break
        ops = ins[j][2].split(None, 1)
        if len(ops) < 2:
            continue
        srcs = ops[1].split(",", 1)[1] if "," in ops[1] else ""
        if re.search(r"\b%s\b" % r, srcs):
            print(f"{fn[:40]} {addr}: {txt}  ->  {ins[j][1]}: {ins[j][2]}")
            break
