"""SASS instructions executed per CUDA source line of the stream kernel, normalised
to one RGB-channel pixel of config 2 (calibrated at 5 MUFU per pixel-channel).
usage: ncu_sass_per_px.py src.csv   (ncu --page source --csv --print-source=cuda,sass)"""
import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
sass=[]
cur=None; curfile=None
for r in rows:
    if not r: continue
    if r[0]=='File Path': curfile=r[1].split('/')[-1]; continue
    if r[0] in('Function Name','Line No'): continue
    if r[0].strip(): cur=(curfile,int(r[0])); continue
    if len(r)>7 and r[2].startswith('0x'):
        sass.append((int(r[2],16), r[3].strip(), int(r[7] or 0), cur, int(r[4] or 0)))
sass.sort()
mufu=sum(n for a,t,n,l,s in sass if 'MUFU' in t)
scale = 5.0/ (mufu*32/ (200*3*1024*1024))  # calibrate: 5 MUFU per px-ch
norm = lambda n: n*32/(200*3*1024*1024)*scale
by=collections.defaultdict(int); ops=collections.defaultdict(collections.Counter)
for a,t,n,l,s in sass:
    by[l]+=n
    op=(t.split()[1] if t.startswith('@') else t.split()[0]).split('.')[0]
    ops[l][op]+=n
print('scale',scale,'total per px', norm(sum(by.values())))
for l in sorted(by, key=lambda x:(x[0] or '', x[1])):
    v=norm(by[l])
    if v>=0.3: print(f'{l[0]}:{l[1]:<5} {v:6.2f}  ', ' '.join(f'{o}:{norm(c):.1f}' for o,c in ops[l].most_common(5)))
