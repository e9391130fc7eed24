"""Local search over Gram task layouts (CTF_GRAM_TUNE): per-group chunk
rotation and length, x-row padding and group order, minimising the modelled
shared-memory wavefronts at unchanged FMA work. Usage: search.py NT M L T iters seed."""
import random, sys, json
from bank_model import *
NT,M,L,T,iters=[int(v) for v in sys.argv[1:6]]
random.seed(int(sys.argv[6]) if len(sys.argv)>6 else 0)
gs=groups(M,L); th=alloc(gs,NT); ng=len(gs)
xp0=1048
def ev(st):
    order,rot,cadd,xpk=st
    g2=[gs[i] for i in order]; t2=[th[i] for i in order]
    xw,ww,f=cost(g2,table(g2,t2,T,L,rot,cadd),NT,xp0+xpk)
    return xw+ww,f,(xw,ww)
st=(list(range(ng)),[0]*ng,[0]*ng,0)
best,bf,det=ev(st); f0=bf
print("start",best,bf,det,flush=True)
for it in range(iters):
    order,rot,cadd,xpk=[list(x) if isinstance(x,list) else x for x in st]
    k=random.random()
    if k<0.5: g=random.randrange(ng); rot[g]=random.randrange(32)
    elif k<0.7: g=random.randrange(ng); cadd[g]=random.choice([0,1,2])
    elif k<0.8: xpk=random.randrange(16)
    else:
        i=random.randrange(ng); j=random.randrange(ng)
        if gs[order[i]][4]==gs[order[j]][4]: order[i],order[j]=order[j],order[i]
    c,f,d=ev((order,rot,cadd,xpk))
    if f<=f0*1.005 and c<=best:
        if c<best: print(it,c,f,d,flush=True)
        best=c; st=(order,rot,cadd,xpk)
print(json.dumps({"order":st[0],"rot":st[1],"cadd":st[2],"xpk":st[3],"cost":int(best)}))
