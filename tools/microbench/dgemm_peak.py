"""cuBLAS DGEMM (torch float64 matmul) throughput: the FP64 tensor roofline denominator."""
import json, torch
torch.backends.cuda.matmul.allow_tf32 = False
res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record(); c = a @ b; e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[n] = 2 * n**3 / best / 1e9
    print(f"DGEMM n={n}: {res[n]:.2f} TFLOP/s ({best:.2f} ms)")
# tall-skinny Gram via cuBLAS for reference: A^T A with A = 1M x 200
for (N, m) in ((1 << 20, 200), (1 << 20, 32), (200000, 200)):
    a = torch.randn(N, m, dtype=torch.float64, device="cuda")
    for _ in range(3):
        a.T @ a
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0.record(); c = a.T @ a; e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"cuBLAS Gram N={N} m={m}: {2*N*m*m/best/1e9:.2f} TFLOP/s ({best:.3f} ms)")
json.dump(res, open("gpurun_out/dgemm_peak.json", "w"))
