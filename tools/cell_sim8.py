"""Cell k-NN cost model: distance-1 visits L1-then-R1 (the kernel) vs per-lane nearest side first, and the resulting far-visit queue sizes (development tool, round 2 session 3).  python tools/cell_sim8.py [npairs]"""
import sys, numpy as np
import os; sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from cell_sim7 import lane_scan, pairs_of, K, C
def stats(x,y):
    n=len(x); ncol=(n+C-1)//C
    yr=np.empty(n,np.int64); yr[np.argsort(y,kind='stable')]=np.arange(n)
    cols=[np.arange(c*C,min(n,(c+1)*C))[np.argsort(yr[c*C:min(n,(c+1)*C)],kind='stable')] for c in range(ncol)]
    start_of=lambda c,i: int(np.sum(yr[cols[c]]<(yr[i]//32)*32))
    gapL=lambda i,c: np.float32(x[i]-x[(c+1)*C-1]); gapR=lambda i,c: np.float32(x[c*C]-x[i])
    st=dict(base_d1=0, near_d1=0, base_q=0, near_q=0)
    for w in range(ncol):
        mem=cols[w]; cx,cy=x[mem],y[mem]
        Ls=[]
        for l_,i in enumerate(mem):
            L,s=lane_scan(np.full(K,np.inf,np.float32),x[i],y[i],cx,cy,l_+1,l_-1); Ls.append(L)
        # baseline: L1 then R1 lockstep
        for mode in ('base','near'):
            Lm=[L.copy() for L in Ls]
            if mode=='base':
                for c in (w-1,w+1):
                    if not (0<=c<ncol): continue
                    ms=0
                    for l_,i in enumerate(mem):
                        g=gapL(i,c) if c<w else gapR(i,c)
                        if g<Lm[l_][K-1]:
                            s0=start_of(c,i); cm=cols[c]
                            Lm[l_],s=lane_scan(Lm[l_],x[i],y[i],x[cm],y[cm],s0,s0-1); ms=max(ms,s)
                    st['base_d1']+=ms
            else:
                done=[set() for _ in mem]
                for rnd in range(2):
                    ms=0
                    for l_,i in enumerate(mem):
                        cands=[]
                        for c in (w-1,w+1):
                            if 0<=c<ncol and c not in done[l_]:
                                g=gapL(i,c) if c<w else gapR(i,c)
                                if g<Lm[l_][K-1]: cands.append((g,c))
                        if not cands: continue
                        g,c=min(cands); done[l_].add(c)
                        s0=start_of(c,i); cm=cols[c]
                        Lm[l_],s=lane_scan(Lm[l_],x[i],y[i],x[cm],y[cm],s0,s0-1); ms=max(ms,s)
                    st['near_d1']+=ms
            # count queued lanes
            q=0
            for l_,i in enumerate(mem):
                nl=w-2>=0 and gapL(i,w-2)<Lm[l_][K-1]; nr=w+2<ncol and gapR(i,w+2)<Lm[l_][K-1]
                q+= (nl or nr)
            st[mode+'_q']+=q
    return st
agg={}
for xa,xb in pairs_of(int(sys.argv[1]) if len(sys.argv)>1 else 3):
    if xb.std()>xa.std(): xa,xb=xb,xa
    o=np.argsort(xa,kind='stable'); st=stats(xa[o],xb[o])
    for k,v in st.items(): agg[k]=agg.get(k,0)+v
print(agg)
