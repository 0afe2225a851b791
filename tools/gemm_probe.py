import sys, numpy as np
sys.path.insert(0, '.')
import paper_2201_05500_b200 as kp
M = N = 128; K = 32
for (k0, m0, n0) in [(0, 0, 0), (0, 1, 0), (0, 5, 0), (0, 33, 0), (1, 0, 0), (3, 2, 7), (9, 0, 0), (17, 40, 70)]:
    A = np.zeros((K, M), np.float32); B = np.zeros((K, N), np.float32)
    A[k0, m0] = 1.0; B[k0, n0] = 1.0
    C = kp.gemm_tn(A, B, engine=2)
    nz = np.argwhere(np.abs(C) > 0.5)
    print((k0, m0, n0), "->", nz[:6].tolist(), "n_nonzero", len(nz))
