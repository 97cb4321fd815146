"""Warp-instructions and stall samples per candidate, bucketed by source-line
ranges of engine.h (one bucket per event-loop phase), from an ncu source page
(--page source --csv --print-source cuda,sass).
usage: ncu_phases_lines.py <src.csv> <n_candidates> "<first>:<last>:<name>,..." """
import csv,sys
from collections import defaultdict
def f(x):
    try: return float(x)
    except: return 0.0
path,ncand=sys.argv[1],float(sys.argv[2])
ranges=[(int(a),int(b),n) for a,b,n in (x.split(':') for x in sys.argv[3].split(','))]
hdr=fname=cur=None; seen=set(); agg=defaultdict(lambda:[0.0,0.0])
for r in csv.reader(open(path)):
    if not r: continue
    if r[0]=='File Path': fname=r[1].split('/')[-1]; continue
    if r[0]=='Line No': hdr=r; si=hdr.index('Warp Stall Sampling (All Samples)'); ie=hdr.index('Instructions Executed'); continue
    if hdr is None or r[0]=='Function Name': continue
    if r[0]: cur=(fname,int(r[0])); continue
    if r[2] in seen or r[2]=='...': continue
    seen.add(r[2])
    ph='other:'+cur[0]
    if cur[0]=='engine.h':
        for a,b,n in ranges:
            if a<=cur[1]<=b: ph=n;break
        else: ph='engine.h other'
    agg[ph][0]+=f(r[si]); agg[ph][1]+=f(r[ie])
ts=sum(v[0] for v in agg.values())
for k,v in sorted(agg.items(),key=lambda x:-x[1][0]): print(f"{k:30s} inst/cand={v[1]/ncand:9.0f} samples={100*v[0]/ts:5.1f}%")
