import numpy as np, paper_2201_05500_b200 as kp
for (M,N,K) in [(19456,256,512),(65536,256,6400)]:
    rng=np.random.default_rng(1)
    A=rng.standard_normal((M,K)).astype(np.float32); B=rng.standard_normal((N,K)).astype(np.float32)
    h4=kp.gemm_nt(A,B,engine=4); h4b=kp.gemm_nt(A,B,engine=4); h6=kp.gemm_nt(A,B,engine=6)
    print(M,N,K,'4==4',np.array_equal(h4,h4b))
    d=np.nonzero(np.any(h4!=h6,axis=1))[0]
    print(' rows differ:',len(d), d[:10], d[-10:] if len(d) else None)
    if len(d): 
        t=np.unique(d//256); print(' tiles differ:', t[:20], len(t))
        r=d[0]; c=np.nonzero(h4[r]!=h6[r])[0]; print(' cols', c[:20], len(c), h4[r,c[0]], h6[r,c[0]])
