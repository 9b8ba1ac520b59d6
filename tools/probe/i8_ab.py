"""A/B timing of anomaly-kernel library variants: python i8_ab.py VAR1 VAR2 ... ('' = product build).
Each variant runs in its own process: correctness vs the FP64 DMMA kernel at 2^18 rows,
then the median of 7 launches at 2^24 rows (config-4 size)."""
import os, subprocess, sys, json
CHILD = r'''
import os, sys, ctypes, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1302_3876_b200 import _native
dev = torch.device('cuda', 0); lib = _native.lib(); s = torch.cuda.current_stream().cuda_stream
n = 128
g = torch.Generator(device=dev); g.manual_seed(5)
def run(ns, mode, reps):
    os.environ["ENKF_ANOMALY"] = mode
    x = torch.randn((ns, n), dtype=torch.float64, device=dev, generator=g) * torch.exp(torch.randn((ns, 1), dtype=torch.float64, device=dev, generator=g))
    t = torch.eye(n, dtype=torch.float64, device=dev) + 0.05 * torch.randn((n, n), dtype=torch.float64, device=dev, generator=g)
    out = torch.empty_like(x); plan = _native.Plan(ns, 1, n, 0)
    ts = []
    for i in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); lib.enkf_anomaly_update_f64(plan.handle, x.data_ptr(), t.data_ptr(), out.data_ptr(), ns, s); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return x, t, out, sorted(ts)[len(ts)//2]
g.manual_seed(5); x, t, o8, _ = run(1 << 18, "i8", 2)
g.manual_seed(5); _, _, o64, _ = run(1 << 18, "fp64", 2)
err = ((o8 - o64).abs().max() / o64.abs().max()).item()
_, _, _, ms = run(1 << 24, "i8", 7)
print(json.dumps({"variant": os.environ.get("ENKF_LIB_VARIANT", ""), "err": err, "ms_2e24": ms, "GBps": 2 * (1 << 24) * n * 8 / ms / 1e6}))
'''
for v in (sys.argv[1:] or [""]):
    env = dict(os.environ, ENKF_LIB_VARIANT=v)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    print(r.stdout.strip() or r.stderr[-2000:], flush=True)
