"""Cell k-NN cost model: distance-1 columns scanned one after the other (the kernel) vs JOINTLY (one candidate up and down in both neighbour columns per step): warp scan steps per pair (development tool, round 2 session 3).  python tools/cell_sim10.py"""
import sys, numpy as np
import os; sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from cell_sim7 import lane_scan, pairs_of, K, C, ins
def joint_scan(L, xi, yi, cols_xy, starts):
    # cols_xy: list of (cx,cy) arrays; starts: list of start or None; scan all columns' up/down together
    ptr=[]
    for (cx,cy),s0 in zip(cols_xy,starts):
        if s0 is None: continue
        ptr.append([cx,cy,s0,s0-1,s0<len(cy),s0-1>=0])
    steps=0
    while any(p[4] or p[5] for p in ptr):
        steps+=1
        for p in ptr:
            cx,cy=p[0],p[1]
            if p[4]:
                j=p[2]; d=max(abs(np.float32(xi-cx[j])),abs(np.float32(yi-cy[j]))); L=ins(L,d)
            if p[5]:
                j=p[3]; d=max(abs(np.float32(xi-cx[j])),abs(np.float32(yi-cy[j]))); L=ins(L,d)
        for p in ptr:
            cx,cy=p[0],p[1]
            if p[4]:
                j=p[2]; stop=np.float32(cy[j]-yi)>=L[K-1]; p[2]+=1; p[4]=(not stop) and p[2]<len(cy)
            if p[5]:
                j=p[3]; stop=np.float32(yi-cy[j])>=L[K-1]; p[3]-=1; p[5]=(not stop) and p[3]>=0
    return L,steps
def run(x,y):
    n=len(x); ncol=(n+C-1)//C
    yr=np.empty(n,np.int64); yr[np.argsort(y,kind='stable')]=np.arange(n)
    cols=[np.arange(c*C,min(n,(c+1)*C))[np.argsort(yr[c*C:min(n,(c+1)*C)],kind='stable')] for c in range(ncol)]
    start_of=lambda c,i: int(np.sum(yr[cols[c]]<(yr[i]//32)*32))
    gapL=lambda i,c: np.float32(x[i]-x[(c+1)*C-1]); gapR=lambda i,c: np.float32(x[c*C]-x[i])
    st=dict(base=0,joint=0)
    for w in range(ncol):
        mem=cols[w]; cx,cy=x[mem],y[mem]
        Ls=[]
        for l_,i in enumerate(mem):
            L,s=lane_scan(np.full(K,np.inf,np.float32),x[i],y[i],cx,cy,l_+1,l_-1); Ls.append(L)
        Lb=[L.copy() for L in Ls]
        for c in (w-1,w+1):
            if not(0<=c<ncol): continue
            ms=0
            for l_,i in enumerate(mem):
                g=gapL(i,c) if c<w else gapR(i,c)
                if g<Lb[l_][K-1]:
                    s0=start_of(c,i); cm=cols[c]
                    Lb[l_],s=lane_scan(Lb[l_],x[i],y[i],x[cm],y[cm],s0,s0-1); ms=max(ms,s)
            st['base']+=ms
        ms=0
        for l_,i in enumerate(mem):
            L=Ls[l_].copy(); cxy=[];starts=[]
            for c in (w-1,w+1):
                if not(0<=c<ncol): continue
                g=gapL(i,c) if c<w else gapR(i,c)
                cm=cols[c]; cxy.append((x[cm],y[cm])); starts.append(start_of(c,i) if g<L[K-1] else None)
            L,s=joint_scan(L,x[i],y[i],cxy,starts); ms=max(ms,s)
        st['joint']+=ms
    return st
agg={}
for xa,xb in pairs_of(3):
    if xb.std()>xa.std(): xa,xb=xb,xa
    o=np.argsort(xa,kind='stable'); s=run(xa[o],xb[o])
    for k,v in s.items(): agg[k]=agg.get(k,0)+v/3
print(agg)
