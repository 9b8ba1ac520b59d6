"""One-off box probe: host cores/RAM, cuBLAS DGEMM (torch.matmul fp64) at the
anomaly-update shape and 8192^3, and H2D/D2H pinned copy bandwidth."""
import json
import os
import subprocess
import time

import torch

out = {}
out["cpu_count"] = os.cpu_count()
out["affinity"] = len(os.sched_getaffinity(0))
try:
    out["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
except Exception:
    pass
out["mem_total_gib"] = int(open("/proc/meminfo").readline().split()[1]) / 2**20
free, total = torch.cuda.mem_get_info()
out["gpu_free_gib"] = free / 2**30
out["gpu_total_gib"] = total / 2**30


def best_ms(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
ms = best_ms(lambda: a @ b)
out["dgemm_8192_tflops"] = 2 * 8192**3 / ms / 1e9
del a, b
x = torch.randn(2**24, 128, dtype=torch.float64, device="cuda")
t = torch.randn(128, 128, dtype=torch.float64, device="cuda")
ms = best_ms(lambda: x @ t)
out["dgemm_anomaly_cfg4_ms"] = ms
out["dgemm_anomaly_cfg4_tflops"] = 2 * 2**24 * 128 * 128 / ms / 1e9
y = torch.empty_like(x)
ms = best_ms(lambda: torch.addmm(x, x, t, out=y))
out["addmm_anomaly_cfg4_ms"] = ms
ms = best_ms(lambda: y.copy_(x))
out["copy_f64_cfg4_gbs"] = 2 * x.numel() * 8 / ms / 1e6
v = torch.randn(2**20, 128, dtype=torch.float64, device="cuda")
ms = best_ms(lambda: v.T @ v)
out["gram_vtv_cfg4_ms"] = ms
out["gram_vtv_cfg4_tflops"] = 2 * 2**20 * 128 * 128 / ms / 1e9
del x, y, v
h = torch.empty(2**28, dtype=torch.float64).pin_memory()
d = torch.empty(2**28, dtype=torch.float64, device="cuda")
t0 = time.perf_counter(); d.copy_(h); torch.cuda.synchronize(); t1 = time.perf_counter()
d.copy_(h); torch.cuda.synchronize(); t2 = time.perf_counter()
out["h2d_pinned_gbs"] = 2**31 / (t2 - t1) / 1e9
h.copy_(d); torch.cuda.synchronize(); t3 = time.perf_counter()
out["d2h_pinned_gbs"] = 2**31 / (t3 - t2) / 1e9
try:
    out["nvidia_smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.sm,clocks.max.sm,power.limit", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
except Exception as e:  # noqa
    out["nvidia_smi"] = str(e)
print(json.dumps(out))
