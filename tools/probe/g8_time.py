"""Run the int8 Gram a few times (for ncu launch lists): python g8_time.py [log2_obs] [log2_state]"""
import sys, torch
sys.path.insert(0, '.')
from paper_1302_3876_b200 import _native
lg_o = int(sys.argv[1]) if len(sys.argv) > 1 else 18
lg_s = int(sys.argv[2]) if len(sys.argv) > 2 else 21
dev = torch.device('cuda', 0); lib = _native.lib(); s = torch.cuda.current_stream().cuda_stream
n, ns, no = 128, 1 << lg_s, 1 << lg_o
x = torch.randn((ns, n), dtype=torch.float64, device=dev)
idx = torch.sort(torch.randperm(ns, device=dev)[:no]).values
y = torch.randn((no, n), dtype=torch.float64, device=dev)
r = 0.25 + 0.75 * torch.rand((no,), dtype=torch.float64, device=dev)
plan = _native.Plan(ns, no, n, 0)
gram = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)
for i in range(3):
    lib.enkf_ism_gram_f64(plan.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(), gram.data_ptr(), s)
torch.cuda.synchronize()
print("ok")
