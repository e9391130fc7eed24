"""Shared-memory bank model of gram_kernel's Gram loads (x products: 8-byte loads
processed per half-warp over 16 bank pairs; weights: 4-byte loads over 32
banks), validated against ncu on cfg1 (x 4128 vs 4145 wavefronts per CTA,
weights 2064 vs 1961). cost() returns (x wavefronts, weight wavefronts, FMA
warp-instructions) of a task table built like build_gram_table()."""
import random, sys
import numpy as np
def groups(M,L):
    gs=[]
    for m in range(M):
        for m2 in range(m,M):
            for d in range(0 if m==m2 else -(L-1), L):
                alo=max(-(L-1),-(L-1)-d); ahi=min(L-1,L-1-d)
                gs.append((m,m2,d,alo,ahi-alo+1))
    return sorted(gs,key=lambda g:-g[4])
def alloc(gs,NT):
    ng=len(gs); total=sum(g[4] for g in gs)
    th=[1]*ng; used=ng; want=[NT*g[4]/total for g in gs]
    while used<NT:
        bd=-1e30;best=0
        for g in range(ng):
            if want[g]-th[g]>bd: bd=want[g]-th[g];best=g
        th[best]+=1;used+=1
    return th
def table(gs,th,T,L,rot=None,cadd=None):
    U0=-(L-1); ln=T+2*(L-1); tab=[]
    for g in range(len(gs)):
        wn=th[g]; clen=(((ln+wn-1)//wn)|1) + (2*cadd[g] if cadd else 0); n=(ln+clen-1)//clen
        ch=[(U0+i*clen,U0+min(ln,(i+1)*clen)) for i in range(n)]
        r=rot[g]%n if rot else 0
        ch=ch[r:]+ch[:r]
        for i in range(wn):
            tab.append((g,)+ch[i] if i<n else (-1,0,0))
    return tab
def cost(gs,tab,NT,xp,UB=4,NS=2):
    xw=0; ww=0; fma=0
    for w0 in range(0,NT,32):
        lanes=[(l,)+tab[w0+l] for l in range(32)]
        act=[(l,g,u0,u1) for (l,g,u0,u1) in lanes if g>=0]
        if not act: continue
        nb=np.array([(u1-u0+UB-1)//UB for l,g,u0,u1 in act])
        cmax=max(gs[g][4] for l,g,u0,u1 in act)
        fma+=nb.max()*UB*(2+NS*cmax)
        ln=np.array([l for l,g,u0,u1 in act]); s0=np.array([u0 for l,g,u0,u1 in act])
        r1=np.array([gs[g][0]*xp for l,g,u0,u1 in act])+s0
        r2=np.array([gs[g][1]*xp+gs[g][2] for l,g,u0,u1 in act])+s0
        rw=np.array([-gs[g][3] for l,g,u0,u1 in act])+s0
        for s in range(nb.max()):
            a=nb>s
            for i in range(UB):
                off=s*UB+i
                for r in (r1,r2):
                    for h in (0,1):
                        sel=a&((ln//16)==h)
                        if sel.any():
                            v=np.unique(r[sel]+off)
                            xw+=np.bincount(v%16,minlength=16).max()
                v=np.unique(rw[a]+off)
                ww+=NS*np.bincount(v%32,minlength=32).max()
    return xw,ww,fma
if __name__=="__main__":
    NT,M,L,T=[int(v) for v in sys.argv[1:5]]
    gs=groups(M,L); th=alloc(gs,NT)
    base=cost(gs,table(gs,th,T,L),NT,1048 if (M,L)==(2,5) else 0)
    print("base",base)
