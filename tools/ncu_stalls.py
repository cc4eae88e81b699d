"""Per CUDA source line stall-reason breakdown from an ncu source page
(--page source --csv --print-source=cuda,sass).
usage: ncu_stalls.py file.csv [file-substring] [topN]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
hdr = None
cur_file = None
agg = defaultdict(lambda: defaultdict(float))
text = {}
line = None
reasons = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        reasons = [(i, h[6:]) for i, h in enumerate(hdr)
                   if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None:
        continue
    if r[0].strip():
        try:
            line = (cur_file, int(r[0]))
        except ValueError:
            continue
        text[line] = r[1]
        for i, n in reasons:  # CUDA line rows carry the aggregated values
            try:
                agg[line][n] += float(r[i] or 0)
            except ValueError:
                pass
tot = defaultdict(float)
for l, d in agg.items():
    for n, v in d.items():
        tot[n] += v
T = sum(tot.values())
print("overall:", ", ".join(f"{n} {100 * v / T:.1f}%" for n, v in
                            sorted(tot.items(), key=lambda x: -x[1]) if v / T > 0.01))
lines = sorted(agg, key=lambda l: -sum(agg[l].values()))
for l in lines[:top]:
    if want and want not in (l[0] or ""):
        continue
    d = agg[l]
    s = sum(d.values())
    parts = ", ".join(f"{n} {v / s * 100:.0f}%" for n, v in sorted(d.items(), key=lambda x: -x[1])
                      if v / s > 0.08)
    print(f"{(l[0] or '').split('/')[-1]}:{l[1]:<4} {100 * s / T:5.1f}%  [{parts}]  {text[l].strip()[:60]}")
