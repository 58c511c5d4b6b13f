"""Probe: cuBLAS DGEMM (torch.matmul float64) and copy bandwidth on this B200 -> JSON line."""
import json, torch, time
torch.backends.cuda.matmul.allow_tf32 = False
res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"dgemm_{n}_tflops"] = 2 * n**3 / best / 1e9
# tall-skinny shapes like the hot path
for (m, k, nn) in ((1023, 2046, 256), (4095, 8190, 128), (2047, 4094, 512)):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda"); b = torch.randn(k, nn, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize(); best = 1e9
    for _ in range(20):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"dgemm_{m}x{k}x{nn}_us"] = best * 1e3
    res[f"dgemm_{m}x{k}x{nn}_tflops"] = 2 * m * k * nn / best / 1e9
print(json.dumps(res))
