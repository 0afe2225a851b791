import sys, numpy as np
sys.path.insert(0, '.')
import paper_2201_05500_b200 as kp
for (M, N, K) in [(128, 128, 32), (300, 256, 6400), (65, 40, 100)]:
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32); B = rng.standard_normal((N, K)).astype(np.float32)
    want = A.astype(np.float64) @ B.astype(np.float64).T
    tc = kp.gemm_nt(A, B, engine=2)
    simt = kp.gemm_nt(A, B, engine=1)
    tc2 = kp.gemm_nt(A, B, engine=2)
    print(M, N, K, "tc", np.abs(tc - want).max() / np.sqrt(K), "simt", np.abs(simt - want).max() / np.sqrt(K), "tc2", np.abs(tc2 - want).max() / np.sqrt(K))
