"""Launch only the int8 anomaly kernel (for ncu captures): python i8_only.py [log2_rows] [launches]."""
import os, sys
import torch
sys.path.insert(0, '.')
from paper_1302_3876_b200 import _native
dev = torch.device('cuda', 0)
lib = _native.lib()
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 22
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n, ns = 128, 1 << lg
x = torch.randn((ns, n), dtype=torch.float64, device=dev)
t = torch.eye(n, dtype=torch.float64, device=dev) + 0.01 * torch.randn((n, n), dtype=torch.float64, device=dev)
out = torch.empty_like(x)
plan = _native.Plan(ns, 1, n, 0)
s = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(reps):
    if i == reps - 1:
        e0.record()
    lib.enkf_anomaly_update_f64(plan.handle, x.data_ptr(), t.data_ptr(), out.data_ptr(), ns, s)
e1.record()
torch.cuda.synchronize()
print("last launch ms", e0.elapsed_time(e1), "GB/s", 2 * ns * n * 8 / e0.elapsed_time(e1) / 1e6)
