"""Per-source-line instruction and stall-sample shares of one ncu report.

    python scripts/ncu_lines.py report.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, errors="replace").stdout
hdr = None
line = None
fname = None
src = {}
inst = collections.Counter()
stall = collections.Counter()
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    d = dict(zip(hdr, r))
    if r[0].strip():
        try:
            line = (fname, int(r[0]))
            src[line] = r[1]
        except ValueError:
            pass
    try:
        inst[line] += int(d.get("Instructions Executed") or 0)
        stall[line] += int(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        pass
ti = sum(inst.values()) or 1
ts = sum(stall.values()) or 1
print("warp instructions", ti, "stall samples", ts)
for k, v in sorted(inst.items(), key=lambda kv: -kv[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100 * v / ti:5.1f}%inst {100 * stall[k] / ts:5.1f}%stall {k[0]}:{k[1]} {src.get(k, '').strip()[:90]}")
