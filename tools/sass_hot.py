"""Hot SASS of an ncu report (source page, SASS view): instructions executed
per contiguous address region, plus the top instructions.
Usage: sass_hot.py <sass.csv> [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ia], 16), r[isrc], int(float(r[iex] or 0)), int(float(r[isamp] or 0))))
    except (ValueError, IndexError):
        pass
tot = sum(d[2] for d in data)
tots = sum(d[3] for d in data)
print(f"total warp instructions {tot:.4g}, samples {tots}")
# regions: consecutive instructions with the same execution count
regions = []
cur = None
for a, s, n, sm in data:
    if cur and cur[2] == n:
        cur[1] = a
        cur[3] += 1
        cur[4] += sm
        cur[5].append(s)
    else:
        cur = [a, a, n, 1, sm, [s]]
        regions.append(cur)
regions.sort(key=lambda r: -r[2] * r[3])
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for a0, a1, n, cnt, sm, srcs in regions[:top]:
    ops = {}
    for s in srcs:
        op = s.split()[0] if s.split() else "?"
        if op.startswith("@"):
            op = s.split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    opstr = " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:8])
    print(f"{a0:6x}-{a1:6x} x{n:>11d} len {cnt:4d} -> {100 * n * cnt / tot:5.1f}% inst  {100 * sm / max(tots, 1):5.1f}% samp  {opstr}")
