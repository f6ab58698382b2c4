import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; cur_file = None; cur_line = None; src = {}
stall = collections.Counter(); inst = collections.Counter()
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur_file = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None or r[0] == 'Function Name': continue
    if r[0] != '':
        cur_line = (cur_file, int(r[0])); src[cur_line] = r[1]
        d = dict(zip(hdr[4:], r[4:]))
        try:
            stall[cur_line] += int(d.get('Warp Stall Sampling (All Samples)', 0) or 0)
            inst[cur_line] += int(d.get('Instructions Executed', 0) or 0)
        except ValueError: pass
tot = sum(stall.values()); toti = sum(inst.values())
print("total samples", tot, "inst", toti)
for k, v in stall.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    print(f"{100*v/tot:5.1f}% {100*inst[k]/max(toti,1):5.1f}%i {k[0]}:{k[1]:5d} {src[k].strip()[:90]}")
