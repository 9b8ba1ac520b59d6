import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import reduced_model as M
from paper_1302_3876_b200 import _native
dev = torch.device('cuda', 0)
lib = _native.lib()
s = torch.cuda.current_stream().cuda_stream
for ws in ('0', '1'):
    os.environ['ENKF_DISABLE_WS'] = ws
    for n in (2, 3, 4, 8, 16, 20, 64, 96, 128):
        for nobs in (5, 50, 1000):
            g = np.random.default_rng(n * 1000 + nobs)
            r = g.uniform(0.5, 2, nobs); v = g.standard_normal((nobs, n)); d = g.standard_normal((nobs, n))
            plan = _native.Plan(0, nobs, n, 0)
            z = torch.empty((nobs, n), dtype=torch.float64, device=dev)
            a = torch.empty((n, n), dtype=torch.float64, device=dev)
            rt, vt, dt = (torch.from_numpy(t).to(dev) for t in (r, v, d))
            st = _native.EnkfStatus()
            rc = lib.enkf_ism_solve_f64(plan.handle, rt.data_ptr(), vt.data_ptr(), dt.data_ptr(), z.data_ptr(), a.data_ptr(), s, ctypes.byref(st))
            gram = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)
            gm = M.gram_solve(v, d, r)
            zm, am = M.solve(r, v, d)
            ez = np.abs(z.cpu().numpy() - zm).max() / np.abs(zm).max()
            ea = np.abs(a.cpu().numpy() - am).max() / np.abs(am).max()
            print(f"disable_ws={ws} n={n} nobs={nobs} rc={rc} errZ={ez:.2e} errA={ea:.2e}", flush=True)
