"""Which source functions occupy the warm band of the instruction footprint
(128-byte lines ranked by executed instructions: band = cumulative share
between LO and HI).  Input: ncu --page source --csv --print-source cuda,sass.

    python scripts/icache_bands.py cs.csv [LO HI]
"""
import collections
import csv
import re
import sys

import os
src = open(os.environ.get("ARROW_SRC", "paper_2505_11916_b200/csrc/sim_core.cuh")).read().split("\n")
defs = []
for i, l in enumerate(src, 1):
    m = re.match(r"\s*(?:AS_HD|AS_NOINL AS_HD|static AS_HD)\s+[\w:<>&\*\s]+?\b(\w+)\(", l)
    if m:
        defs.append((i, m.group(1)))


def fof(n):
    best = "?"
    for i, name in defs:
        if i <= n:
            best = name
        else:
            break
    return best


fname, line = None, None
ins = []
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0].strip():
        try:
            line = int(r[0])
        except ValueError:
            pass
        continue
    try:
        a = int(r[2], 16)
        e = int(r[7] or 0)
    except (ValueError, IndexError):
        continue
    fn = fof(line) if fname == "sim_core.cuh" else fname
    ins.append((a, e, fn))
base = min(a for a, _, _ in ins)
lines = collections.defaultdict(lambda: [0, collections.Counter()])
for a, e, fn in ins:
    L = lines[(a - base) // 128]
    L[0] += e
    L[1][fn] += 1
tot = sum(v[0] for v in lines.values())
lo, hi = (float(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (0.9, 0.999)
acc = 0
band = collections.Counter()
band_exec = collections.Counter()
nl = 0
for k, (e, fns) in sorted(lines.items(), key=lambda kv: -kv[1][0]):
    prev = acc
    acc += e
    if prev >= lo * tot and prev < hi * tot:
        nl += 1
        for fn, c in fns.items():
            band[fn] += c * 16
            band_exec[fn] += e * c / sum(fns.values())
print(f"band {lo:.3f}-{hi:.3f}: {nl} lines = {nl * 128 / 1024:.1f} KB, {100 * sum(band_exec.values()) / tot:.2f}% of executed")
for fn, b in band.most_common(30):
    print(f"{b / 1024:6.2f} KB  {100 * band_exec[fn] / tot:6.3f}% exec  {fn}")
