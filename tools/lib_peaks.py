"""Harness-only library references: cuBLAS DGEMM and TF32 SGEMM throughput via torch (not the product path)."""
import json, time, torch
def bench(dtype, n, tf32=False, secs=4.0):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype); b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(5):
        e0.record(); a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    t0 = time.time(); it = 0; e0.record()
    while time.time() - t0 < secs:
        a @ b; it += 1
        if it % 8 == 0: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize(); sus = e0.elapsed_time(e1) / it
    f = 2 * n ** 3
    return f / best / 1e9, f / sus / 1e9
r = {}
r["cublas_dgemm_8192_burst_tflops"], r["cublas_dgemm_8192_sustained_tflops"] = bench(torch.float64, 8192)
r["cublas_dgemm_4096_burst_tflops"], _ = bench(torch.float64, 4096, secs=0.5)
r["cublas_tf32_8192_burst_tflops"], r["cublas_tf32_8192_sustained_tflops"] = bench(torch.float32, 8192, tf32=True)
print(json.dumps(r))
