import sys, numpy as np
sys.path.insert(0, '.')
import paper_2201_05500_b200 as kp
def nt(M, N, K):
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32); B = rng.standard_normal((N, K)).astype(np.float32)
    want = A.astype(np.float64) @ B.astype(np.float64).T
    tc = kp.gemm_nt(A, B, engine=2)
    print("nt", M, N, K, np.abs(tc - want).max() / np.sqrt(K))
def tn(M, N, K):
    rng = np.random.default_rng(M * N + K)
    A = rng.standard_normal((K, M)).astype(np.float32); B = rng.standard_normal((K, N)).astype(np.float32)
    want = A.astype(np.float64).T @ B.astype(np.float64)
    tc = kp.gemm_tn(A, B, engine=2)
    print("tn", M, N, K, np.abs(tc - want).max() / np.sqrt(K))
for step in sys.argv[1:]:
    kind, shp = step.split(':')
    M, N, K = map(int, shp.split(','))
    (nt if kind == 'nt' else tn)(M, N, K)
