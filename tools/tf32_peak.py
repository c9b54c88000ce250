"""Measured dense TF32 tensor throughput on this B200 (context for the Pearson block roofline,
whose prescribed peak is the measured bf16 peak x the nominal tf32:bf16 ratio 0.5): cuBLAS via
torch.matmul with TF32 enabled, 8192^3 fp32 operands, best of 10 (burst) and back to back for 4 s
(sustained).  Development tool; prints one JSON line."""
import json
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
N = 8192
a = torch.randn(N, N, device="cuda")
b = torch.randn(N, N, device="cuda")
c = torch.empty(N, N, device="cuda")
flop = 2 * N ** 3
for _ in range(3):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
best = 0.0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    best = max(best, flop / (e0.elapsed_time(e1) / 1e3) / 1e12)
t = time.time()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
k = 0
while time.time() - t < 4.0:
    for _ in range(20):
        torch.matmul(a, b, out=c)
    k += 20
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sust = k * flop / (e0.elapsed_time(e1) / 1e3) / 1e12
print(json.dumps({"tf32_tflops_burst": best, "tf32_tflops_sustained": sust, "n": N, "how": "torch.matmul fp32 with allow_tf32 (cuBLAS)"}))
