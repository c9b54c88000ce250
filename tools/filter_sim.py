"""Filter-test variants of the KSG sweep's outer chunks (development tool; DESIGN.md §10
"Tried and rejected").  Replays the CTA kernel's schedule (32-member warps, exact own block and
adjacent chunks, filtered groups of 4 outward) on C4 pairs and counts, per filtered group, whether
the warp vote triggers the merge network under
  ex: the exact test  min_j max(|dx|, |dy|) < l[k-1]   (what the kernel does), and
  dy: a cheaper conservative test  min_j |dy| < l[k-1]  (no x distance, no per-j max).
  h16: a packed-f16 test on per-pair centred, power-of-two-scaled values with a threshold
       inflated by the rounding bound (conservative, so eps stays exact).
ALU cost model: ex = 7 per group + 16 per trigger; dy = 3 per group + 20 per trigger;
h16 = 5 per group (2 HMNMX2 |.|-max, 1 HMNMX2 min, cross-half min, compare) + 21 per trigger.

    python tools/filter_sim.py [npairs]
"""
import sys, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sweep_sim as S
K=3; G=4
def run(npairs=6):
    tot = {"ex":[0,0,0.0], "dy":[0,0,0.0], "h16":[0,0,0.0]}
    for xa, xb in S.pairs_of(npairs):
        if xb.std() > xa.std(): xa, xb = xb, xa
        o = np.argsort(xa, kind="stable"); x, y = xa[o], xb[o]; n=len(x)
        cx, cy = np.float32(np.median(x)), np.float32(np.median(y))
        R = max(np.abs(x-cx).max(), np.abs(y-cy).max()); sc = 2.0**(14-np.ceil(np.log2(R)))
        hx = ((x-cx).astype(np.float32)*sc).astype(np.float16).astype(np.float64)/sc
        hy = ((y-cy).astype(np.float32)*sc).astype(np.float16).astype(np.float64)/sc
        slack = R*sc*2**-9/sc
        for b0 in range(0, n, 32):
            mem = np.arange(b0, min(b0+32, n)); nm=len(mem)
            xi, yi = x[mem], y[mem]
            def dist(js):
                d = np.maximum(np.abs(xi[:,None]-x[None,js]), np.abs(yi[:,None]-y[None,js])); d[mem[:,None]==js[None,:]]=np.inf; return d
            def ins(L, v): return np.sort(np.concatenate([L, v],1),1)[:, :K]
            L = ins(np.full((nm,K),np.inf), dist(mem))
            b1 = min(b0+32,n); nlo, nhi = (b0+31)//32, (n-b1+31)//32
            for mode in ("ex","dy","h16"):
                LL = L.copy(); st={0:(0 if nlo else -1),1:(0 if nhi else -1)}; first={0:True,1:True}
                while st[0]>=0 or st[1]>=0:
                    for dr in (0,1):
                        c=st[dr]
                        if c<0: continue
                        js = np.arange(max(0,b0-(c+1)*32), b0-c*32) if dr==0 else np.arange(b1+c*32, min(n,b1+(c+1)*32))
                        t=LL[:,K-1]
                        need = np.any(xi - x[js[-1]] < t) if dr==0 else np.any(x[js[0]]-xi < t)
                        if not need: st[dr]=-1; continue
                        d=dist(js); dyy=np.abs(yi[:,None]-y[None,js])
                        if first[dr]: LL=ins(LL,d)
                        else:
                            order = np.arange(len(js))[::-1] if dr==0 else np.arange(len(js))
                            for g in range(0,len(js),G):
                                cols=order[g:g+G]
                                tot[mode][0]+=1
                                if mode=="ex": test = d[:,cols].min(1) < LL[:,K-1]
                                elif mode=="dy": test = dyy[:,cols].min(1) < LL[:,K-1]
                                else:
                                    hd = np.maximum(np.abs(hx[mem][:,None]-hx[None,js[cols]]), np.abs(hy[mem][:,None]-hy[None,js[cols]])).astype(np.float32)
                                    T = (1+2**-10)*(LL[:,K-1]*(1+2**-22) + slack) + 2**-23
                                    test = hd.min(1) < T
                                if np.any(test):
                                    tot[mode][1]+=1; LL=ins(LL,d[:,cols])
                        first[dr]=False
                        st[dr]= c+1 if c+1 < (nlo if dr==0 else nhi) else -1
    for m in tot:
        g,t,_=tot[m]; print(m, "groups", g, "triggered", t, "frac %.3f"%(t/g))
    gh,th,_=tot["h16"]; print("packed-f16 filter ALU cost:", 5*gh+21*th)
    ge,te,_=tot["ex"]; gd,td,_=tot["dy"]
    print("ALU cost exact filter:", 7*ge+16*te, " dy filter:", 3*gd+20*td, " ratio %.3f"%((3*gd+20*td)/(7*ge+16*te)))
run(int(sys.argv[1]) if len(sys.argv)>1 else 6)
