"""SAH cost of the greedy largest-area 4-wide collapse (k_collapse_level)
against the SAH-optimal collapse (dynamic programming over slots) of the
same binary tree; usage: python tools/collapse_sah.py SCENE [C_node]."""
import sys, time, numpy as np
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_19977_b200 import build_bvh
from workloads import scene_by_name
name = sys.argv[1] if len(sys.argv) > 1 else 'pushbutton'
sc = scene_by_name(name)
t0=time.time(); bvh = build_bvh(sc.triangles, device=None); print('build', time.time()-t0)
L, R, C = bvh.left_child, bvh.right_child, bvh.triangle_count
lo, hi = bvh.bounds_min, bvh.bounds_max
ext = hi - lo
A = ext[:,0]*ext[:,1] + ext[:,1]*ext[:,2] + ext[:,2]*ext[:,0]
N = len(L)
CN, CT = float(sys.argv[2]) if len(sys.argv)>2 else 1.5, 1.0
# greedy collapse (as k_collapse_level)
def greedy():
    cost = 0.0; roots=[0]; nw=0
    while roots:
        nxt=[]
        for r in roots:
            nw+=1
            cost += A[r]*CN
            ch=[L[r],R[r]]
            while len(ch)<4:
                best=-1; ba=-1
                for k,c in enumerate(ch):
                    if C[c]==0 and A[c]>ba: ba=A[c]; best=k
                if best<0: break
                x=ch[best]; ch[best:best+1]=[L[x],R[x]]
            for c in ch:
                if C[c]==0: nxt.append(c)
                else: cost += A[c]*C[c]*CT
        roots=nxt
    return cost/A[0], nw
# DP: S[n][j] j=1..4, process in decreasing index (children > parent)
INF=1e300
S=np.full((N,5),INF); D=np.full((N,5),INF)
for n in range(N-1,-1,-1):
    if C[n]>0:
        S[n,1:]=A[n]*C[n]*CT
        continue
    l,r=L[n],R[n]
    for k in range(2,5):
        D[n,k]=min(S[l,j]+S[r,k-j] for j in range(1,k))
    W=A[n]*CN+D[n,4]
    S[n,1]=W
    for j in range(2,5):
        S[n,j]=min(S[n,j-1],D[n,j])
print('greedy SAH', greedy(), 'DP optimal', (A[0]*CN+D[0,4])/A[0])
