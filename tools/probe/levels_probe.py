"""Time the levels kernel alone (enkf_ism_levels_f64) on a realistic Gram.

    python tools/probe/levels_probe.py [N, default 128]
"""
import ctypes, json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1302_3876_b200 import _native
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dev = torch.device("cuda", 0)
g = np.random.Generator(np.random.Philox(3))
v = g.standard_normal((4096, n)) / np.sqrt(n - 1)
d = g.standard_normal((4096, n))
gram = np.concatenate([v.T @ v, v.T @ d / np.sqrt(n - 1)], axis=1)
gd = torch.from_numpy(gram).to(dev)
a = torch.empty((n, n), dtype=torch.float64, device=dev); t = torch.empty_like(a)
plan = _native.Plan(1, 1, n, 0)
lib = _native.lib(); s = torch.cuda.current_stream().cuda_stream
for _ in range(10): lib.enkf_ism_levels_f64(plan.handle, gd.data_ptr(), a.data_ptr(), t.data_ptr(), None, s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100): lib.enkf_ism_levels_f64(plan.handle, gd.data_ptr(), a.data_ptr(), t.data_ptr(), None, s)
e1.record(); torch.cuda.synchronize()
ref = np.linalg.solve(np.eye(n) + gram[:, :n], gram[:, n:])
print(json.dumps({"n": n, "levels_us": e0.elapsed_time(e1) / 100 * 1e3, "A_err": float(np.abs(a.cpu().numpy() - ref).max() / np.abs(ref).max())}))
if os.environ.get("ENKF_LIB_VARIANT") == "lvt":
    buf = (ctypes.c_longlong * (20 * 6))()
    lib_raw = ctypes.CDLL(_native.LIB_PATH)
    lib_raw.enkf_debug_lv_trace(buf)
    tr = np.array(buf[:]).reshape(20, 6)
    t0 = tr[0, 0]
    nb = (n + 7) // 8
    for b in range(nb):
        ph = tr[b, :4] - t0
        nxt = (tr[b + 1, 0] if b < nb - 1 else tr[16, 0]) - t0
        print(b, "gather->LDL", ph[1] - ph[0], "LDL", ph[2] - ph[1], "solve", ph[3] - ph[2], "update", nxt - ph[3])
    print("epilogue start", tr[16, 0] - t0)
