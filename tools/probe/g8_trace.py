"""Per-stage trace of gram_i8_kernel CTA 0 (needs the "g8trace" variant: -DG8_TRACE_ON)."""
import ctypes, os, sys
import numpy as np, torch
os.environ.setdefault("ENKF_LIB_VARIANT", "g8trace")
sys.path.insert(0, '.')
from paper_1302_3876_b200 import _native
dev = torch.device('cuda', 0); lib = _native.lib(); s = torch.cuda.current_stream().cuda_stream
n, ns, no = 128, 1 << 21, 1 << 18
x = torch.randn((ns, n), dtype=torch.float64, device=dev)
idx = torch.sort(torch.randperm(ns, device=dev)[:no]).values
y = torch.randn((no, n), dtype=torch.float64, device=dev)
r = 0.25 + 0.75 * torch.rand((no,), dtype=torch.float64, device=dev)
plan = _native.Plan(ns, no, n, 0)
gram = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)
for i in range(3):
    lib.enkf_ism_gram_f64(plan.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(), gram.data_ptr(), s)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (512 * 12))()
fn = lib.enkf_debug_g8_trace; fn.argtypes = [ctypes.c_void_p]
assert fn(ctypes.addressof(buf)) == 0
tr = np.array(buf, dtype=np.float64).reshape(512, 12)
t0 = tr[0, 0]
tr = np.where(tr > 0, (tr - t0) / 1000.0, np.nan)
print("stage: issued  saw  means  stored")
for st in list(range(0, 10)) + list(range(200, 210)):
    print(st, " ".join(f"{tr[st, k]:8.2f}" for k in range(4)))
print("block: mma start, issued")
for b in list(range(0, 6)) + list(range(50, 56)):
    print(b, f"{tr[b, 8]:8.2f} {tr[b, 9]:8.2f}")
st = np.arange(40, 300)
for a, b_, lab in [(0, 1, "issue->saw"), (1, 2, "saw->means"), (2, 3, "means->stored")]:
    v = tr[st, b_] - tr[st, a]
    print(f"{lab:16s} mean {np.nanmean(v):7.2f} us")
print("stage interval", np.nanmean(np.diff(tr[st, 3])), "us")
