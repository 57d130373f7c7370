#!/usr/bin/env python
"""Per-CUDA-line work of an ncu --set full capture, normalised per work unit:
instructions, L1 shared-memory wavefronts (and the ideal count), global L1
tag requests and the share of warp-stall samples.

    python tools/ncu_lines.py <rep> <units> [top] [sort-column 0..4]

units = work units in the captured launch (e.g. 32-row units of a fact pass).
"""
import csv,io,sys,subprocess
rep=sys.argv[1]; units=float(sys.argv[2])
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(io.StringIO(out)))
agg={}
fname='?';hdr=None
for r in rows:
    if not r: continue
    if r[0]=='File Path': fname=r[1].split('/')[-1]; continue
    if r[0]=='Line No': hdr=r; idx={h:i for i,h in enumerate(r)}; continue
    if r[0]=='Function Name' or hdr is None: continue
    if r[0]!='':
        key=(fname,r[0],r[1][:70])
        def f(n):
            try: return float(r[idx[n]] or 0)
            except: return 0.0
        a=agg.setdefault(key,[0,0,0,0,0]); a[0]+=f('L1 Wavefronts Shared'); a[1]+=f('L1 Tag Requests Global'); a[2]+=f('L1 Wavefronts Shared Ideal'); a[3]+=f('Instructions Executed'); a[4]+=f('Warp Stall Sampling (All Samples)')
tot=[sum(v[i] for v in agg.values()) for i in range(5)]
print('per unit: shared wf %.1f  global tags %.1f  inst %.1f'%(tot[0]/units,tot[1]/units,tot[3]/units))
for k,v in sorted(agg.items(), key=lambda kv:-(kv[1][int(sys.argv[4]) if len(sys.argv)>4 else 4]))[:int(sys.argv[3]) if len(sys.argv)>3 else 30]:
    print('%-12s %4s stall%% %5.1f inst %6.1f sh %5.1f(%5.1f) gtag %5.1f  %s'%(k[0][:12],k[1],100*v[4]/tot[4],v[3]/units,v[0]/units,v[2]/units,v[1]/units,k[2]))
