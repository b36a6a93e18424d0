"""Where a kernel's time goes, from an ncu `--page source --csv` export (SASS rows).

usage: ncu -i rep.ncu-rep --page source --csv > src.csv
       python tools/ncu_source_breakdown.py src.csv [lo_addr hi_addr]

Prints the main loop's (the backward branch with the densest VIADDMNMX body) share of
warp-stall samples and executed instructions, the top 1 KB address buckets outside it,
and the stall-reason mix; with an address range, the per-instruction listing.
"""
import csv,sys,re,collections
rows=list(csv.reader(open(sys.argv[1])))
h=rows[1]; data=rows[2:]
ia=h.index("Address"); isrc=h.index("Source"); isamp=h.index("Warp Stall Sampling (All Samples)"); iex=h.index("Instructions Executed")
stall_cols=[i for i,c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
ins=[]
for r in data:
    try: a=int(r[ia],16)
    except: continue
    ins.append((a,r[isrc],float(r[isamp] or 0),float(r[iex] or 0),{h[i]:float(r[i] or 0) for i in stall_cols}))
# main loop: backward branch with highest VIADDMNMX density
loops=[]
for a,t,_,_,_ in ins:
    m=re.search(r'BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)',t)
    if m:
        tgt=int(m.group(1),16)
        if tgt<a:
            sub=[x for b,x,_,_,_ in ins if tgt<=b<=a]
            loops.append((sum('VIADDMNMX' in x for x in sub)/len(sub),tgt,a))
loops.sort(reverse=True); _,lo,hi=loops[0]
tot_s=sum(x[2] for x in ins); tot_e=sum(x[3] for x in ins)
in_s=sum(x[2] for x in ins if lo<=x[0]<=hi); in_e=sum(x[3] for x in ins if lo<=x[0]<=hi)
print(f"main loop {hex(lo)}-{hex(hi)}: samples {in_s/tot_s:.3f}, inst {in_e/tot_e:.3f}; total inst {tot_e:.3e}")
# walk-like instructions anywhere (VIADDMNMX/VIMNMX3/IMAD.IADD) share
walk=sum(x[3] for x in ins if re.match(r'\s*(VIADDMNMX|VIMNMX3|IMAD\.IADD)',x[1]))
print(f"walk-op share of executed inst: {walk/tot_e:.3f}")
# top sample regions outside loop in 64-instruction buckets
bk=collections.Counter(); bke=collections.Counter()
for a,t,s,e,_ in ins:
    if not(lo<=a<=hi): bk[a//0x400]+=s; bke[a//0x400]+=e
for b,s in bk.most_common(8): print(hex(b*0x400), f"samples {s/tot_s:.3f} inst {bke[b]/tot_e:.3f}")
st=collections.Counter()
for x in ins:
    for k,v in x[4].items(): st[k]+=v
print({k:round(v/tot_s,3) for k,v in st.most_common(8)})
if len(sys.argv)>2:
    lo2=int(sys.argv[2],16); hi2=int(sys.argv[3],16)
    for a,t,s,e,stl in ins:
        if lo2<=a<hi2:
            top=max(stl.items(),key=lambda kv:kv[1])
            print(hex(a)[-5:], f"{s:7.0f} {e:10.0f}", t[:70], top[0] if s>0 else '')
