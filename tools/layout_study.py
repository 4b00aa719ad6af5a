"""Cluster-layout study (cluster efficiency): for a water box, the pruned
list's tile count, entry count and cluster efficiency (pairs inside rc / 32 per tile) of
alternative slab layouts -- column cross-section for `cell` atoms per cube, then three halvings
of each 32-atom slab along the given axes (j clusters after two, i clusters after three).
libnbx's layout is cell 32, axes (y, x, z).  Full periodic list, both orders of every pair.

    python tools/layout_study.py [natoms]
"""
import sys, numpy as np
sys.path.insert(0,'/root/repo')
from scipy.spatial import cKDTree
from paper_2405_01420_b200 import systems
n=int(sys.argv[1]) if len(sys.argv)>1 else 30000
s=systems.make('water12m', n)
box=s.box.astype(np.float64); x=np.mod(s.x.astype(np.float64), box)
N=x.shape[0]; dens=N/np.prod(box)
t=cKDTree(x,boxsize=box)
pairs=t.query_pairs(1.02,output_type='ndarray')
d=x[pairs[:,0]]-x[pairs[:,1]]; d-=box*np.round(d/box); r2=(d*d).sum(1)
useful=2*(r2<1.0).sum()
def split(g, axes):
    if not axes: return [g]
    o=g[np.argsort(x[g,axes[0]],kind='stable')]
    h=len(o)//2
    return split(o[:h],axes[1:])+split(o[h:],axes[1:])
def run(cell_atoms, axes):
    cs=np.cbrt(cell_atoms/dens); nx=max(1,int(np.floor(box[0]/cs+0.5))); ny=max(1,int(np.floor(box[1]/cs+0.5)))
    cx=np.minimum((x[:,0]/box[0]*nx).astype(int),nx-1); cy=np.minimum((x[:,1]/box[1]*ny).astype(int),ny-1)
    col=cx*ny+cy
    order=np.lexsort((x[:,2],col))
    icl=np.empty(N,int); jcl=np.empty(N,int)
    ic=0; jc=0
    cols=col[order]
    starts=np.r_[0,np.nonzero(np.diff(cols))[0]+1,N]
    for a,b in zip(starts[:-1],starts[1:]):
        idx=order[a:b]
        for s0 in range(0,len(idx),32):
            sc=idx[s0:s0+32]
            groups4=split(sc,axes) if len(sc)==32 else [sc[k:k+4] for k in range(0,32,4)]
            for k,g in enumerate(groups4):
                icl[g]=ic+k; jcl[g]=jc+k//2
            ic+=8; jc+=4
    a=np.r_[icl[pairs[:,0]],icl[pairs[:,1]]]; b=np.r_[jcl[pairs[:,1]],jcl[pairs[:,0]]]
    key=np.unique(a.astype(np.int64)*10**7+b)
    tiles=key.size
    ents=np.unique((key//10**7)//8*10**7+key%10**7).size
    cost=ents*35+tiles*35
    print(f"cell {cell_atoms:4d} axes {axes}: tiles {tiles:8d} entries {ents:8d} t/e {tiles/ents:.2f} eff {useful/(32*tiles):.3f} cost {cost/1e6:.2f}M", flush=True)
for cell,axes in [(32,(1,0,2)),(64,(0,1,2)),(64,(1,0,2)),(64,(0,1,0)),(128,(0,1,0)),(16,(1,2,2)),(32,(2,1,0)),(48,(1,0,2)),(64,(2,0,1))]:
    run(cell,axes)
