import sys, numpy as np
sys.path.insert(0, '.')
import paper_2201_05500_b200 as kp
shapes = [tuple(map(int, s.split(','))) for s in sys.argv[1:]]
for (M, N, K) in shapes:
    rng = np.random.default_rng(1)
    A = rng.standard_normal((M, K)).astype(np.float32); B = rng.standard_normal((N, K)).astype(np.float32)
    want = A.astype(np.float64) @ B.astype(np.float64).T
    tc = kp.gemm_nt(A, B, engine=2)
    e = np.abs(tc - want) / np.sqrt(K)
    bad = e > 1e-3
    print(M, N, K, "err", e.max(), "bad rows", np.unique(np.where(bad)[0])[:8], "bad cols", np.unique(np.where(bad)[1])[:8], "frac bad", bad.mean())
