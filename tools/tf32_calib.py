import torch, time
torch.backends.cuda.matmul.allow_tf32 = True
dev = 'cuda'
def t(M, N, K, reps=10):
    a = torch.randn(M, K, device=dev); b = torch.randn(K, N, device=dev)
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"tf32 {M}x{N}x{K}: {ms:.3f} ms {2*M*N*K/ms/1e9:.0f} TF/s")
t(8192, 8192, 8192)
t(65536, 256, 6400)
t(65536, 6400, 256)
t(256, 6400, 65536)
torch.backends.cuda.matmul.allow_tf32 = False
t(8192, 8192, 8192, 3)
