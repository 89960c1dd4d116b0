"""Per-SASS-instruction hot spots from `ncu -i X --page source --csv --print-source sass` output.
usage: python tools/sass_hot.py export.csv [min_inst] [kernel-substring]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 300000
want = sys.argv[3] if len(sys.argv) > 3 else ""
sec = []
for r in rows:
    if r and r[0] == "Kernel Name":
        sec.append([r[1], None, []])
    elif r and r[0] == "Address":
        sec[-1][1] = r
    elif sec and sec[-1][1] is not None:
        sec[-1][2].append(r)
seen = set()
for name, hdr, data in sec:
    if want not in name or name in seen:
        continue
    seen.add(name)
    ie, st, at = (hdr.index(k) for k in ("Instructions Executed", "Warp Stall Sampling (All Samples)", "Avg. Threads Executed"))
    data = [r for r in data if len(r) > ie and r[ie].isdigit()]
    tot = sum(int(r[ie]) for r in data)
    print(f"== {name[:90]}  total warp inst {tot}")
    for i, r in enumerate(data):
        if int(r[ie]) >= thr or int(r[st]) >= 200:
            print(f"{i:4d} {int(r[ie]):>10} {int(r[st]):>6} {r[at]:>5}  {r[1].strip()[:90]}")
