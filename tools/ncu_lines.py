"""Aggregate an ncu source page (--print-source=cuda,sass --csv) per CUDA line:
instructions executed and stall samples.  usage: ncu_lines.py file.csv [file-substring]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else ""
cur_file, hdr = None, None
inst, stall, text = defaultdict(int), defaultdict(int), {}
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0].strip():
        line = (cur_file, int(r[0]))
        text[line] = r[1]
    if len(r) > 7 and r[2]:
        try:
            inst[line] += int(r[7] or 0)
            stall[line] += int(r[4] or 0)
        except ValueError:
            pass
ti, ts = sum(inst.values()), sum(stall.values())
print(f"total inst {ti}  stall samples {ts}")
key = (lambda k: -inst[k]) if "--by-inst" in sys.argv else (lambda k: -stall[k])
for k in sorted(inst, key=key)[:40]:
    if want and want not in k[0]:
        continue
    print(f"{k[0].split('/')[-1]:>18}:{k[1]:<4} inst {100*inst[k]/ti:5.1f}%  stall {100*stall[k]/ts:5.1f}%  {text[k].strip()[:80]}")
