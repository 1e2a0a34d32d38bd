"""Bank-conflict search for the element kernel's volume layout.

U(a1, a2, a3) sits at a1 S1 + a2 S2 + a3 S3 (element stride VS) and is touched by three
half-warp access patterns (64-bit accesses, 16 banks of 8 bytes): the phase-1 store over
(a2, a3), the y-reduction loads over (a1, a3) and the z-reduction loads over (a1, a2).  This
script enumerates strides and paddings and prints the layouts with the fewest wavefronts, next
to the layout the kernel uses.  For odd N no linear layout reaches the ideal count.

    python tools/bank_search.py N
"""
import sys, itertools
def cost(N,S1,S2,S3,VS,G,NT):
    NQ=N*N; tot=[0,0,0]
    for hw in range(0,NT,16):
        lanes=[t for t in range(hw,hw+16) if t<G*NQ]
        if not lanes: continue
        for pat in range(3):
            banks={}
            for t in lanes:
                e=t//NQ;q=t%NQ;qa=q//N;qb=q%N
                if pat==0: addr=e*VS+qa*S2+qb*S3
                elif pat==1: addr=e*VS+qa*S1+qb*S3
                else: addr=e*VS+qa*S1+qb*S2
                banks.setdefault(addr%16,set()).add(addr)
            tot[pat]+=max(len(v) for v in banks.values())
    return tot
def inj(N,S1,S2,S3):
    s={a*S1+b*S2+c*S3 for a in range(N) for b in range(N) for c in range(N)}
    return len(s)==N**3
N=int(sys.argv[1]); NQ=N*N; G=256//NQ; NT=(G*NQ+31)//32*32
ideal=(G*NQ+15)//16*3
res=[]
for S3 in range(1,8):
  for S2 in range(1,NQ+12):
    for S1 in range(1,N*NQ+20):
        ext=(N-1)*(S1+S2+S3)+1
        if ext>N**3*1.6+8: continue
        if not inj(N,S1,S2,S3): continue
        for vp in range(0,16):
            VS=ext+vp
            t=cost(N,S1,S2,S3,VS,G,NT)
            res.append((sum(t),t,S1,S2,S3,VS))
res.sort()
print("N",N,"G",G,"ideal",ideal,"current",cost(N,NQ,N,1,N*NQ,G,NT))
for r in res[:6]: print(r)
