"""cuBLAS DGEMM on the step's tall-skinny shapes (development reference point)."""
import torch
N = 109268
torch.backends.cuda.matmul.allow_tf32 = False
for (a, b) in [(200, 200), (164, 100), (64, 200), (100, 100), (32, 200), (64, 64), (32, 32)]:
    A = torch.randn(N, a, dtype=torch.float64, device="cuda")
    B = torch.randn(N, b, dtype=torch.float64, device="cuda")
    for _ in range(3):
        C = A.T @ B
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        C = A.T @ B
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 * 1e3
    print(f"cublas gram {a}x{b} N={N}: {t:7.1f} us {2*N*a*b/t/1e6:6.2f} TF", flush=True)
for (a, b) in [(200, 200), (200, 100), (64, 200), (100, 100), (32, 200), (164, 32)]:
    A = torch.randn(N, a, dtype=torch.float64, device="cuda")
    Cm = torch.randn(a, b, dtype=torch.float64, device="cuda")
    for _ in range(3):
        O = A @ Cm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        O = A @ Cm
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 * 1e3
    print(f"cublas nn {a}x{b} N={N}: {t:7.1f} us {2*N*a*b/t/1e6:6.2f} TF", flush=True)
