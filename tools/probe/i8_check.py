"""Compare the tcgen05 int8-digit anomaly update with the FP64 DMMA kernel."""
import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_1302_3876_b200 import _native, workloads as W
import reduced_model as M

dev = torch.device('cuda', 0)
lib = _native.lib()
s = torch.cuda.current_stream().cuda_stream
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 10
p = W.config4(scale)
ns, nobs, n = p.shape
x = torch.from_numpy(p.x).to(dev)
# T from the model (same as the levels kernel up to rounding)
a, _ = M.levels(M.gram_analysis(p.x[p.indices], p.perturbed, p.r))
T = torch.from_numpy(np.ascontiguousarray(M.transform(a))).to(dev)
outs = {}
for mode in ("fp64", "i8"):
    os.environ["ENKF_ANOMALY"] = mode
    plan = _native.Plan(ns, nobs, n, 0)
    out = torch.full_like(x, float('nan'))
    rc = lib.enkf_anomaly_update_f64(plan.handle, x.data_ptr(), T.data_ptr(), out.data_ptr(), ns, s)
    torch.cuda.synchronize()
    st = _native.EnkfStatus()
    rc2 = lib.enkf_plan_sync_status(plan.handle, s, ctypes.byref(st))
    outs[mode] = out.cpu().numpy()
    # timing
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        lib.enkf_anomaly_update_f64(plan.handle, x.data_ptr(), T.data_ptr(), out.data_ptr(), ns, s)
    e1.record(); torch.cuda.synchronize()
    print(mode, "rc", rc, rc2, "ms/launch", e0.elapsed_time(e1) / 5, flush=True)
ref = p.x @ M.transform(a)
f, q = outs["fp64"], outs["i8"]
print("fp64 vs numpy", np.abs(f - ref).max() / np.abs(ref).max())
d = np.abs(q - f)
print("i8 vs fp64 max rel", np.nanmax(d) / np.abs(f).max(), "nan count", np.isnan(q).sum())
if np.nanmax(d) / np.abs(f).max() > 1e-9 or np.isnan(q).any():
    bad = np.argwhere(~(d <= 1e-9 * np.abs(f).max()))
    print("bad count", len(bad), "first", bad[:10].tolist())
    rows = np.unique(bad[:, 0]); cols = np.unique(bad[:, 1])
    print("bad rows (mod 128) hist", np.bincount(rows % 128, minlength=128)[:32], "ncols", len(cols))
    print("sample q", q[bad[0][0], :8], "f", f[bad[0][0], :8])
