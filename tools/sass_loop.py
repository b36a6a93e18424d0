"""Opcode histogram of a kernel's main loop in `cuobjdump -sass` output.

usage: python tools/sass_loop.py kernel.sass <mangled function name> [x]

The main loop is the backward branch with the densest VIADDMNMX body; with a third
argument, the instructions other than the walk (VIADDMNMX / VIMNMX3 / IMAD.IADD) are listed.
"""
import re,sys,collections
sass=open(sys.argv[1]).read()
fn=sys.argv[2]
i=sass.index("Function : "+fn); j=sass.find("Function : ",i+10); body=sass[i:j if j>0 else None]
ins=[]
for m in re.finditer(r'/\*([0-9a-f]{4,5})\*/\s+([^;]+);',body):
    ins.append((int(m.group(1),16),m.group(2).strip()))
loops=[]
for k,(a,t) in enumerate(ins):
    m=re.search(r'BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)',t)
    if m:
        tgt=int(m.group(1),16)
        if tgt<a:
            sub=[x for b,x in ins if tgt<=b<=a]
            v=sum(1 for x in sub if 'VIADDMNMX' in x)
            loops.append((v/len(sub),len(sub),tgt,a))
loops.sort(reverse=True)
_,n,lo,hi=loops[0]
c=collections.Counter()
for a,t in ins:
    if lo<=a<=hi:
        op=t.split()[0]
        if op.startswith('@'): op=t.split()[1]
        c[op.split('.')[0] if not op.startswith('IMAD') else op]+=1
print(fn[:60],'loop',hex(lo),hex(hi),'n',n)
print(' '.join(f'{k}:{v}' for k,v in c.most_common()))
if len(sys.argv)>3:
    for a,t in ins:
        if lo<=a<=hi and not re.match(r'(VIADDMNMX|VIMNMX3|IMAD.IADD)',t): print('   ',t)
