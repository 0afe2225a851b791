import numpy as np, paper_2201_05500_b200 as kp
for (M,N,K) in [(128,128,32),(128,128,256),(128,128,1024),(128,128,6400),(300,256,256),(300,256,1024),(300,256,6400),(256,128,6400)]:
    rng=np.random.default_rng(1)
    A=rng.standard_normal((M,K)).astype(np.float32); B=rng.standard_normal((N,K)).astype(np.float32)
    want=A.astype(np.float64)@B.astype(np.float64).T
    tc=kp.gemm_nt(A,B,engine=2); si=kp.gemm_nt(A,B,engine=1)
    e=np.abs(tc-want)
    print(M,N,K,"tc",e.max()/np.sqrt(K),"simt",np.abs(si-want).max()/np.sqrt(K), "rows with big err", np.unique(np.where(e>e.max()/4)[0])[:10], "cols", np.unique(np.where(e>e.max()/4)[1])[:10])
