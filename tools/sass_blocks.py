"""Largest straight-line SASS blocks of a kernel with their opcode mix
(static check of the fast sweep step before spending GPU time).
usage: python tools/sass_blocks.py file.sass [nblocks]"""
import re
import sys
from collections import Counter

lines = [l for l in open(sys.argv[1]) if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
blocks, cur = [], []
for l in lines:
    ins = l.split("*/", 1)[1].split(";")[0].strip()
    cur.append(ins)
    if re.search(r"\b(BRA|EXIT|RET|BRX|CALL)\b", ins):
        blocks.append(cur)
        cur = []
blocks.append(cur)
blocks.sort(key=len, reverse=True)
for b in blocks[: int(sys.argv[2]) if len(sys.argv) > 2 else 3]:
    c = Counter(re.sub(r"^@!?U?P\w+\s+", "", i).split()[0].split(".")[0] for i in b)
    print(len(b), dict(c.most_common(25)))
