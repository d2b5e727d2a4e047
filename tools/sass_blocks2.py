"""Static SASS basic blocks of one kernel (cuobjdump -sass), largest first,
with an opcode histogram.  Usage: sass_blocks2.py <obj/.so> <kernel-substring> [n]"""
import re
import subprocess
import sys
from collections import Counter

obj, name = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
body = next(f for f in funcs if name in f.split("\n")[0])
lines = [l for l in body.split("\n") if re.search(r"/\*[0-9a-f]{4,}\*/", l)]
ins = []
for l in lines:
    m = re.search(r"/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
targets = set()
for a, t in ins:
    m = re.search(r"BRA.*?(0x[0-9a-f]+)", t)
    if m:
        targets.add(int(m.group(1), 16))
blocks, cur = [], []
for a, t in ins:
    if a in targets and cur:
        blocks.append(cur)
        cur = []
    cur.append((a, t))
    if re.match(r"(@!?U?P\d\s+)?(BRA|EXIT|RET|BRX|JMP)", t):
        blocks.append(cur)
        cur = []
if cur:
    blocks.append(cur)
print(f"{len(ins)} instructions, {len(blocks)} blocks")
for b in sorted(blocks, key=len, reverse=True)[:n]:
    ops = Counter()
    for _, t in b:
        op = t.split()[0]
        if op.startswith("@"):
            op = t.split()[1]
        ops[op.split(".")[0]] += 1
    print(f"{b[0][0]:6x} len {len(b):4d}: " + " ".join(f"{k}:{v}" for k, v in ops.most_common(14)))
