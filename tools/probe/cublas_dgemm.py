import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = 5 if n < 16384 else 3
    e0.record()
    for _ in range(reps): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cuBLAS DGEMM n={n}: {2*n**3/ms/1e9:.2f} TFLOP/s ({ms:.1f} ms)")
# QR via cusolver (torch.linalg.qr) for context
n = 16384
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
torch.linalg.qr(a[:4096, :4096]); torch.cuda.synchronize()
t = time.perf_counter(); q, r = torch.linalg.qr(a); torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"cusolver geqrf+orgqr n={n}: {dt:.3f} s, {(8/3)*n**3/dt/1e12:.2f} TFLOP/s")
