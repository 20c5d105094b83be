"""Executed warp-instructions per SASS opcode of the four C4 kernels, from ncu
source-page CSV exports (ncu -i rep --page source --csv --print-source sass
--launch-skip k --launch-count 1 > sass_k.csv), in millions.

    python tools/sass_opcode_mix.py DIR   (DIR/sass_0.csv .. sass_3.csv)
"""
import csv, sys, re
from collections import Counter
def mix(path):
    rows=list(csv.reader(open(path)))
    h=rows[1]; ie=h.index('Instructions Executed'); src=h.index('Source'); st=h.index('Warp Stall Sampling (All Samples)')
    c=Counter(); s=Counter(); tot=0
    for r in rows[2:]:
        if len(r)<=ie: continue
        m=re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_.]+)', r[src])
        if not m: continue
        op=m.group(2)
        try: n=int(r[ie] or 0)
        except ValueError: continue
        c[op]+=n; tot+=n
        s[op]+=int(r[st] or 0) if r[st].isdigit() else 0
    return c,s,tot
names=['K1 fwd','K2 fwd','K2 inv','K1 inv']
res=[mix(f'{sys.argv[1]}/sass_{k}.csv') for k in range(4)]
ops=sorted(set().union(*[r[0] for r in res]), key=lambda o:-res[1][0][o])
print('%-24s'%'op', ''.join('%14s'%n for n in names))
for o in ops[:40]:
    print('%-24s'%o, ''.join('%14.1f'%(r[0][o]/1e6) for r in res))
print('%-24s'%'TOTAL', ''.join('%14.1f'%(r[2]/1e6) for r in res))
