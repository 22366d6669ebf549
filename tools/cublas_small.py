"""Harness-only reference: cuBLAS DGEMM (torch.matmul, fp64) at the config-2 and Table-3 sizes,
as a fraction of the measured DMMA peak (37.161 TF/s) -- context for the fp64 engine's small-d
efficiency (tools/time_f64_sk.py measures the engine the same way: mean of back-to-back launches)."""
import json
import torch

PEAK = 37.161
out = {}
for n in (500, 768, 1024, 1536, 2048, 4096):
    a = torch.randn(n, n, device="cuda", dtype=torch.float64)
    b = torch.randn(n, n, device="cuda", dtype=torch.float64)
    c = torch.empty_like(a)
    for _ in range(5):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    it = max(20, int(2e12 / (2 * n ** 3)))
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it):
        torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    tf = 2 * n ** 3 / ms / 1e9
    out[n] = {"ms": round(ms, 5), "tflops": round(tf, 2), "frac_dmma": round(tf / PEAK, 3)}
print(json.dumps({"cublas_dgemm_back_to_back": out}))
