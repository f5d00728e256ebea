"""Warp-stall samples and executed instructions of the 3D face kernels by phase
(source-line attribution; line ranges of faces3d.cuh at the round-2 final commit; dev tool).
usage: ncu -i REPORT --page source --csv --print-source cuda,sass > /tmp/src_all.csv;
       python tools/ncu_phases3d.py 'k_faces3d<(int)1, (int)1'
"""
import csv, sys, collections, os
rows=list(csv.reader(open(os.environ.get('SRC','/tmp/src_all.csv'))))
kname=sys.argv[1]
func=None; path=None; hdr=None
agg=collections.Counter(); samp=collections.Counter(); stl=collections.defaultdict(collections.Counter)
def phase(f, ln):
    if f=='faces3d.cuh':
        if ln<242: return 'prologue/index'
        if ln<355: return '1a window'
        if ln<390: return '1b roe/eigen'
        if ln<424: return 'barrier1'
        if ln<479: return '3 assembly'
        if ln<505: return 'loop'
        if ln<596: return '2a vectors+proj'
        if ln<597: return 'barrier a'
        if ln<620: return '2b field'
        return 'barrier b'
    if f=='physics.cuh':
        if ln>=650: return '2b TENO'
        return 'physics-other'
    if f.startswith('flux3'): return '1b roe/eigen'
    return 'other:'+f
for r in rows:
    if not r: continue
    if r[0]=='File Path': path=r[1].split('/')[-1]; continue
    if r[0]=='Function Name': func=r[1]; continue
    if r[0]=='Line No': hdr=r; continue
    if func is None or kname not in func or hdr is None: continue
    try: ln=int(r[0])
    except: continue
    ph=phase(path,ln)
    try:
        agg[ph]+=int(r[7]); samp[ph]+=int(r[6])
        for i,h in enumerate(hdr):
            if h.startswith('stall_') and '(Not' not in h and r[i] not in ('','-'): stl[ph][h[6:]]+=int(r[i])
    except: pass
ti=sum(agg.values()); ts=sum(samp.values())
for k,v in samp.most_common():
    print(f"{k:16s} inst {100*agg[k]/ti:5.1f}%  samples {100*v/ts:5.1f}%  {', '.join(f'{o}:{100*c/ts:.1f}' for o,c in stl[k].most_common(4))}")
