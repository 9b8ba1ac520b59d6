"""int8 tensor-core Gram vs the FP64 DMMA Gram: python g8_check.py [log2_obs] [log2_state] [heavy]"""
import ctypes, os, subprocess, sys, json
CHILD = r'''
import os, sys, ctypes, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1302_3876_b200 import _native
lg_o, lg_s, heavy = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dev = torch.device('cuda', 0); lib = _native.lib(); s = torch.cuda.current_stream().cuda_stream
n, ns, no = 128, 1 << lg_s, 1 << lg_o
g = torch.Generator(device=dev); g.manual_seed(7)
mu = torch.randn((ns, 1), dtype=torch.float64, device=dev, generator=g)
sig = 0.5 + 1.5 * torch.rand((ns, 1), dtype=torch.float64, device=dev, generator=g)
x = mu + sig * torch.randn((ns, n), dtype=torch.float64, device=dev, generator=g)
idx = torch.sort(torch.randperm(ns, device=dev, generator=g)[:no]).values
y = x[idx].mean(dim=1, keepdim=True) + torch.randn((no, n), dtype=torch.float64, device=dev, generator=g)
if heavy:
    y[no // 3, 5] = 1e6  # far outside the sampled scale -> FP64 fallback
r = 0.25 + 0.75 * torch.rand((no,), dtype=torch.float64, device=dev, generator=g)
plan = _native.Plan(ns, no, n, 0)
gram = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)
st = _native.EnkfStatus()
lib.enkf_plan_reset_status(plan.handle, s)
ts = []
for i in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); rc = lib.enkf_ism_gram_f64(plan.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(), gram.data_ptr(), s); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
rc2 = lib.enkf_plan_sync_status(plan.handle, s, ctypes.byref(st))
np.save(f"/tmp/gram_{os.environ.get('ENKF_GRAM','fp64')}.npy", gram.cpu().numpy())
print(json.dumps({"mode": os.environ.get("ENKF_GRAM", "fp64"), "rc": rc, "status": rc2, "msg": st.message.decode(), "ms": sorted(ts)[2]}))
'''
args = sys.argv[1:] + ["18", "21", "0"][len(sys.argv) - 1:]
import numpy as np
for mode in ("fp64", "i8"):
    env = dict(os.environ, ENKF_GRAM=mode)
    r = subprocess.run([sys.executable, "-c", CHILD] + args[:3], env=env, capture_output=True, text=True, timeout=300)
    print(r.stdout.strip() or r.stderr[-3000:], flush=True)
a, b = np.load("/tmp/gram_fp64.npy"), np.load("/tmp/gram_i8.npy")
d = np.abs(a - b)
print("VV max rel", d[:, :128].max() / np.abs(a[:, :128]).max(), "VD max rel", d[:, 128:].max() / np.abs(a[:, 128:]).max(),
      "symm err", np.abs(b[:, :128] - b[:, :128].T).max(), "nan", np.isnan(b).sum())
