"""Measures the dense TF32 tensor-core peak of this B200 the way MEASURED_PEAKS.json measures
bf16 (torch.matmul 8192^3, fp32 operands with TF32 allowed, best of 10 = burst; back to back
for 4 s = sustained) and writes profiles/measured_tf32.json, which bench.py uses as the tensor
peak of the TF32 precision mode (MEASURED_PEAKS.json has no TF32 figure)."""
import json
import time
from pathlib import Path

import torch

torch.backends.cuda.matmul.allow_tf32 = True
N = 8192
a = torch.randn(N, N, device="cuda")
b = torch.randn(N, N, device="cuda")
c = torch.empty(N, N, device="cuda")
for _ in range(3):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b, out=c)
    e1.record()
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
flop = 2.0 * N ** 3
t0, n = time.perf_counter(), 0
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.perf_counter() - t0 < 4.0:
    for _ in range(10):
        torch.matmul(a, b, out=c)
    n += 10
    torch.cuda.synchronize()
e1.record()
e1.synchronize()
out = {"tf32_tflops": flop / (best / 1e3) / 1e12,
       "tf32_tflops_sustained": flop * n / (e0.elapsed_time(e1) / 1e3) / 1e12,
       "gpu_name": torch.cuda.get_device_name(), "torch": torch.__version__,
       "how": "torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS TF32 tensor cores): best of 10 "
              "(burst) and back to back for 4 s (sustained)"}
Path(__file__).resolve().parent.parent.joinpath("profiles", "measured_tf32.json").write_text(
    json.dumps(out, indent=1))
print(json.dumps(out))
