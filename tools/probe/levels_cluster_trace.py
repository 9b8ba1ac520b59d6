import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1302_3876_b200 import _native
n = int(sys.argv[1])
dev = torch.device("cuda", 0)
g = np.random.Generator(np.random.Philox(3))
v = g.standard_normal((4096, n)) / np.sqrt(n - 1); d = g.standard_normal((4096, n))
gram = np.concatenate([v.T @ v, v.T @ d / np.sqrt(n - 1)], axis=1)
gd = torch.from_numpy(gram).to(dev)
a = torch.empty((n, n), dtype=torch.float64, device=dev); t = torch.empty_like(a)
plan = _native.Plan(1, 1, n, 0); lib = _native.lib(); s = torch.cuda.current_stream().cuda_stream
for _ in range(5): lib.enkf_ism_levels_f64(plan.handle, gd.data_ptr(), a.data_ptr(), t.data_ptr(), None, s)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (20 * 6))()
ctypes.CDLL(_native.LIB_PATH).enkf_debug_lv_trace(buf)
tr = np.array(buf[:]).reshape(20, 6); t0 = tr[0, 0]
for b in range((n + 7) // 8):
    ph = tr[b] - t0
    nxt = (tr[b + 1, 0] - t0) if b + 1 < (n + 7) // 8 else float('nan')
    print(b, "gather", ph[1]-ph[0], "LDL", ph[2]-ph[1], "solve", ph[3]-ph[2], "update", ph[4]-ph[3], "push", ph[5]-ph[4], "csync+", nxt-ph[5])
