"""cuBLAS TF32 dense GEMM peak on this B200 (the tf32 / tf32x3 roofline denominator; MEASURED_PEAKS.json
only has bf16).  Same recipe as the driver's bf16 figure: torch.matmul 8192^3 (2 N^3 flop), best of 10
(burst), and back to back for 4 s (sustained).  Writes gpurun_out/tf32_peak.json (copied to profiles/)."""
import json
import os
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
torch.backends.cuda.matmul.allow_tf32 = True
torch.backends.cudnn.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
c = torch.empty(n, n, device="cuda")
for _ in range(3):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
burst = 2.0 * n ** 3 / (best * 1e-3) / 1e12
t0 = time.perf_counter()
k = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.perf_counter() - t0 < 4.0:
    for _ in range(10):
        torch.matmul(a, b, out=c)
    k += 10
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sustained = 2.0 * n ** 3 * k / (e0.elapsed_time(e1) * 1e-3) / 1e12
kern = torch.cuda.get_device_name()
out = {"tf32_tflops": burst, "tf32_tflops_sustained": sustained, "gpu": kern,
       "how": "torch.matmul fp32 with allow_tf32 (cuBLAS TF32 tensor cores) 8192^3, 2 N^3 flop: best of 10 "
              "(burst) and back to back for 4 s (sustained)", "torch": torch.__version__}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "tf32_peak.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
