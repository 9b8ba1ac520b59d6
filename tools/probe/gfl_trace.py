"""Role timeline of the fused Gram kernel (group 0), profiling build -DGFL_TRACE_ON:
    python tools/build_variant.py gflt -DGFL_TRACE_ON; ENKF_LIB_VARIANT=gflt python tools/probe/gfl_trace.py [scale]"""
import ctypes, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1302_3876_b200 import _native
from paper_1302_3876_b200 import workloads as W
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 0
dev = torch.device("cuda", 0)
d = W.device_problem_shard(5, 1, 0, dev, scale_log2=scale)
x, y, idx, r = d["x"], d["perturbed"], d["idx"], d["r"]
ns, no, n = x.shape[0], y.shape[0], x.shape[1]
os.environ["ENKF_GRAM"] = "i8fused"
plan = _native.Plan(ns, no, n, 0)
lib = _native.lib(); s = torch.cuda.current_stream().cuda_stream
gram = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)
for _ in range(2):
    lib.enkf_ism_gram_f64(plan.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(), gram.data_ptr(), s)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4 * 512 * 6))()
ctypes.CDLL(_native.LIB_PATH).enkf_debug_gfl_trace(buf)
tr = np.array(buf[:], dtype=np.float64).reshape(4, 512, 6)
t0 = tr[tr > 0].min()
tr = np.where(tr > 0, (tr - t0) / 1e3, np.nan)  # us
out = {}
for c in range(4):
    sl = tr[c, :, :3]; pr = tr[c, :, 3:]
    out[c] = {"slicer_block_us": float(np.nanmedian(np.diff(sl[:, 2]))), "slicer_ringwait_us": float(np.nanmedian(sl[:, 1] - sl[:, 0])),
              "slicer_work_us": float(np.nanmedian(sl[:, 2] - sl[:, 1])),
              "prod_block_us": float(np.nanmedian(np.diff(pr[:, 1]))), "prod_readywait_us": float(np.nanmedian(pr[:, 1] - pr[:, 0])),
              "copy_land_us": float(np.nanmedian(pr[:, 2] - pr[:, 1]))}
print(json.dumps(out, indent=1))
np.save("gpurun_out/gfl_trace.npy", tr)
for k in list(range(0, 12)) + list(range(200, 212)):
    print(k, " ".join(f"{tr[c, k, e]:9.1f}" for c in range(4) for e in (3, 4, 5)))
