"""Offline probe (CPU, numpy): distinct 128-B lines / 32-B sectors touched per 32-lane
gather instruction of the PageRank tile kernel (256-edge tiles of the degree-sorted CSC),
as laid out now and with each tile's edges sorted by source slot. Measures whether
reordering edges inside a tile could cut the L1 data-pipe wavefronts per gathered edge.

    python tools/sector_probe.py 22
"""
import numpy as np, sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle
S=int(sys.argv[1]) if len(sys.argv)>1 else 22
s,d,_=oracle.rmat(S,16,1,0.57,0.19,0.19,0,True,False)
ids=np.union1d(s,d)
si=np.searchsorted(ids,s); di=np.searchsorted(ids,d)
indeg=np.bincount(di,minlength=ids.size)
order=np.lexsort((np.arange(ids.size), -indeg))   # slot order: in-degree desc, ties by id
slot=np.empty(ids.size,np.int64); slot[order]=np.arange(ids.size)
ss=slot[si]; ds=slot[di]
o=np.lexsort((ss,ds)); ss=ss[o]; ds=ds[o]          # CSC: by dst slot, then src slot
E=ss.size
T=256; nt=E//T
a=ss[:nt*T].reshape(nt,T)
def lines(x, per=16):
    # x: (nt, T) -> count distinct lines per 32-lane group
    g=x.reshape(nt,T//32,32)//per
    g=np.sort(g,axis=2)
    distinct=1+(np.diff(g,axis=2)!=0).sum(axis=2)
    return distinct.sum()/ (nt*T)
print("scale",S,"E",E)
print("wavefronts/edge unsorted (128B lines):", lines(a))
print("sorted within tile:", lines(np.sort(a,axis=1)))
print("32B sectors unsorted:", lines(a,4), "sorted:", lines(np.sort(a,axis=1),4))
