"""Prune shortcut study (round 2): on the outer list after motion, the
fraction of active unmasked tiles a representative pair keeps, a bounding-box test drops,
and that stay ambiguous (need the full 32-pair test).

    python tools/prune_study.py
"""
import sys, numpy as np
sys.path.insert(0,'.')
from oracle import oracle as O
from paper_2405_01420_b200 import systems
s=systems.make('water12m', 60000)
on=O.OracleNonbonded(s); on.search(s.x)
rng=np.random.default_rng(1)
x1=(s.x+rng.uniform(-0.02,0.02,size=s.x.shape)).astype(np.float32)
on.put_x(x1)
g=on.grid.export(); l=on.list.export(0)  # outer list
xq=g['xq'][:,:3].astype(np.float32)
box=s.box.astype(np.float32); rli2=np.float32(s.rlist_inner**2)
sci=l['sci']; cj=l['cj']; pool=l['pool']
ent_sci=np.repeat(sci['sci'], sci['cj_end']-sci['cj_start']); ent_sh=np.repeat(sci['shift'], sci['cj_end']-sci['cj_start'])
idx=np.concatenate([np.arange(a,b) for a,b in zip(sci['cj_start'],sci['cj_end'])])
cjs=cj['cj'][idx]; meta=cj['meta'][idx]; imask=meta&0xff; pidx=meta>>8
tot=0; keep=0; rep_hit=0; bb_drop=0; amb=0; masked=0
for k in range(8):
    act=((imask>>k)&1==1)
    m=act&(pidx==0); masked+=(act&(pidx>0)).sum()
    ci=8*ent_sci[m]+k; sh=ent_sh[m]
    v=(np.stack([(sh%3-1),((sh//3)%3-1),(sh//9-1)],1)*box).astype(np.float32)
    xi=(xq[(4*ci)[:,None]+np.arange(4)]+v[:,None,:]).astype(np.float32)
    xj=xq[(8*cjs[m])[:,None]+np.arange(8)]
    d=(xi[:,:,None,:]-xj[:,None,:,:]).astype(np.float32)
    r2=(d*d).sum(-1)
    kept=(r2<rli2).any((1,2))
    # representative pair: i atom 1 vs j atom 3 (near cluster centres in the sub-sort) -> try best of a few
    rep=(r2[:,1,3]<rli2)|(r2[:,2,4]<rli2)
    # bbox distance
    # filler atoms at -1e5: exclude from bbox
    fi=xi[:,:,0]>-1e4; fj=xj[:,:,0]>-1e4
    big=np.float32(1e30)
    lo_i=np.where(fi[:,:,None],xi,big).min(1); hi_i=np.where(fi[:,:,None],xi,-big).max(1)
    lo_j=np.where(fj[:,:,None],xj,big).min(1); hi_j=np.where(fj[:,:,None],xj,-big).max(1)
    dd=np.maximum(0,np.maximum(lo_i-hi_j,lo_j-hi_i)); bbd2=(dd*dd).sum(1)
    drop=bbd2>(np.sqrt(rli2)+1e-4)**2
    tot+=m.sum(); keep+=kept.sum(); rep_hit+=rep.sum(); bb_drop+=drop.sum(); amb+=(~rep & ~drop).sum()
    assert not (drop & kept).any()
print("unmasked active tiles",tot,"masked",masked)
print("kept frac",keep/tot,"rep-pair resolves",rep_hit/tot,"bbox drops",bb_drop/tot,"ambiguous",amb/tot)
