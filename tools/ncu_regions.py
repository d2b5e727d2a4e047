"""Stall reasons per hot SASS region of an ncu report (source page CSV, SASS
view).  Regions: runs of instructions with equal execution counts.
Usage: ncu_regions.py <sass.csv> [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ir = [hdr.index(h) for h in reasons]
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ia], 16), r[isrc], int(float(r[iex] or 0)), [int(float(r[i] or 0)) for i in ir]))
    except (ValueError, IndexError):
        pass
tot = sum(d[2] for d in data)
totst = [sum(d[3][j] for d in data) for j in range(len(reasons))]
alls = sum(totst)
print("overall samples:", " ".join(f"{reasons[j][6:]}:{100 * totst[j] / alls:.1f}%" for j in range(len(reasons)) if totst[j] > 0.005 * alls))
regions, cur = [], None
for a, s, n, st in data:
    if cur and cur[2] == n:
        cur[1] = a
        cur[3] += 1
        cur[4] = [x + y for x, y in zip(cur[4], st)]
    else:
        cur = [a, a, n, 1, list(st)]
        regions.append(cur)
regions.sort(key=lambda r: -sum(r[4]))
for a0, a1, n, cnt, st in regions[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    s = sum(st)
    top = sorted(range(len(reasons)), key=lambda j: -st[j])[:5]
    print(f"{a0 & 0xfffff:6x} len {cnt:4d} x{n:>10d} {100 * n * cnt / tot:5.1f}% inst {100 * s / alls:5.1f}% samp | "
          + " ".join(f"{reasons[j][6:]}:{100 * st[j] / max(s, 1):.0f}%" for j in top))
