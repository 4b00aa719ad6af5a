"""Cluster-efficiency study on the oracle's inner list (round 2): fraction of
computed pair slots inside rc, tiles with no pair inside rc, and empty 4 x 4 half tiles.

    python tools/cluster_efficiency.py [config] [natoms]
"""
import sys, numpy as np
sys.path.insert(0,'.')
from oracle import oracle as O
from paper_2405_01420_b200 import systems
s=systems.make(sys.argv[1] if len(sys.argv)>1 else 'water12m', int(sys.argv[2]) if len(sys.argv)>2 else 60000)
on=O.OracleNonbonded(s); on.search(s.x)
g=on.grid.export(); l=on.list.export(1)
xq=g['xq'][:,:3].astype(np.float64)
box=s.box.astype(np.float64)
sci=l['sci']; cj=l['cj']; pool=l['pool']
rc2=s.rc**2
tiles=0; pairs_in=0; empty_tiles=0; half_empty=0; halves=0; slots=0
# vectorize per entry
ent_sci=np.repeat(sci['sci'], sci['cj_end']-sci['cj_start'])
ent_sh=np.repeat(sci['shift'], sci['cj_end']-sci['cj_start'])
# cj entries in order
idx=np.concatenate([np.arange(a,b) for a,b in zip(sci['cj_start'],sci['cj_end'])])
cjs=cj['cj'][idx]; meta=cj['meta'][idx]
imask=meta&0xff; pidx=meta>>8
for k in range(8):
    act=(imask>>k)&1==1
    ci=8*ent_sci[act]+k
    sh=ent_sh[act]
    v=np.stack([(sh%3-1),((sh//3)%3-1),(sh//9-1)],1)*box
    xi=xq[(4*ci)[:,None]+np.arange(4)[None,:]]+v[:,None,:]     # [T,4,3]
    xj=xq[(8*cjs[act])[:,None]+np.arange(8)[None,:]]           # [T,8,3]
    d=xi[:,:,None,:]-xj[:,None,:,:]
    r2=(d*d).sum(-1)                                              # [T,4,8]
    pm=pool[pidx[act]][:,k,0] if True else None
    bits=np.where(pidx[act]>0, pm, 0xffffffff).astype(np.uint64)
    m=((bits[:,None,None]>>(np.arange(4)[None,:,None]*8+np.arange(8)[None,None,:]).astype(np.uint64))&1).astype(bool)
    # filler atoms have coords -1e5 -> far
    inr=(r2<rc2)&m
    tiles+=act.sum(); slots+=32*act.sum()
    pairs_in+=inr.sum()
    empty_tiles+=(inr.reshape(len(inr),-1).sum(1)==0).sum()
    h0=inr[:,:,:4].reshape(len(inr),-1).sum(1)==0
    h1=inr[:,:,4:].reshape(len(inr),-1).sum(1)==0
    half_empty+=h0.sum()+h1.sum(); halves+=2*act.sum()
    # row granularity: i-atoms (4) x 8: empty rows
print(s.name, s.natoms, "entries", len(idx), "tiles", tiles, "tiles/entry", tiles/len(idx))
print("cluster eff", pairs_in/slots, "empty tiles", empty_tiles/tiles, "empty 4x4 halves", half_empty/halves)
print("eff if empty halves skipped", pairs_in/(slots-16*half_empty))
