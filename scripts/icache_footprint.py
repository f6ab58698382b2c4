"""Hot-code footprint of one ncu report: 128-byte instruction lines needed
to cover X% of executed warp instructions (and their stall samples).

    ncu -i rep --page source --csv --print-source sass > sass.csv
    python scripts/icache_footprint.py sass.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, ie, ist = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ins = []
for r in rows[2:]:
    try:
        ins.append((int(r[ia], 16), int(r[ie] or 0), int(r[ist] or 0), r[1].strip()))
    except (ValueError, IndexError):
        pass
base = min(a for a, *_ in ins)
lines = {}
for a, e, s, _ in ins:
    k = (a - base) // 128
    le = lines.setdefault(k, [0, 0])
    le[0] += e
    le[1] += s
tot = sum(v[0] for v in lines.values())
print(f"kernel: {len(ins)} instructions, {len(lines)} lines ({len(lines) * 128 / 1024:.1f} KB)")
acc = 0
srt = sorted(lines.values(), key=lambda v: -v[0])
marks = [0.5, 0.8, 0.9, 0.95, 0.99, 0.999]
for i, (e, s) in enumerate(srt, 1):
    acc += e
    while marks and acc >= marks[0] * tot:
        print(f"{marks[0] * 100:5.1f}% of executed instructions in {i} lines = {i * 128 / 1024:.1f} KB")
        marks.pop(0)
