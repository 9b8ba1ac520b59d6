"""Where config 1's 0.11 ms goes: Python API vs the bare C-ABI call vs kernels."""
import ctypes, json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1302_3876_b200 as P
from paper_1302_3876_b200 import _native, workloads as W
p = W.config1()
dev = torch.device("cuda", 0)
h = P.SelectionOperator.from_indices(p.indices)
x = torch.from_numpy(p.x).to(dev); y = torch.from_numpy(p.perturbed).to(dev); r = torch.from_numpy(p.r).to(dev)
idx = h.device_indices(dev)
obs = P.ObservationBatch(y=None, perturbed=y, perturbations=None)
out = torch.empty_like(x)
plan = _native.get_plan(0, *x.shape[:1], p.perturbed.shape[0], x.shape[1]) if False else _native.get_plan(0, x.shape[0], y.shape[0], x.shape[1])
lib = _native.lib(); s = torch.cuda.current_stream().cuda_stream
res = {}
def bench(fn, reps=2000):
    for _ in range(50): fn()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / reps * 1e6
st = _native.EnkfStatus()
res["python_api_us"] = bench(lambda: P.analysis_step(x, obs, h, r))
res["c_abi_sync_us"] = bench(lambda: lib.enkf_analysis_f64(plan.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(), out.data_ptr(), s, ctypes.byref(st)))
res["c_abi_async_us"] = bench(lambda: lib.enkf_analysis_async_f64(plan.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(), out.data_ptr(), s))
print(json.dumps(res))
