"""Direct launches vs CUDA-graph replay of `enkf_analysis_async_f64` on the small
configs (1-3, launch-latency bound): device ms per step over back-to-back steps
(CUDA events) and host ms per step (wall clock incl. one sync per batch).

    python tools/probe/graph_probe.py [reps]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_1302_3876_b200 import _native  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
dev = torch.device("cuda", 0)
lib = _native.lib()
res = {}
for name, (ns, nobs, n, ident) in {"config1": (40, 20, 20, False), "config2": (4096, 4096, 64, True),
                                   "config3": (16641, 1089, 96, False)}.items():
    rng = np.random.default_rng(ns)
    x = torch.from_numpy(rng.standard_normal((ns, n)) + rng.standard_normal((ns, 1))).to(dev)
    idx = None if ident else torch.from_numpy(np.sort(rng.choice(ns, size=nobs, replace=False))).to(dev)
    hx = x if idx is None else x[idx]
    y = hx.mean(dim=1, keepdim=True) + torch.randn((nobs, n), dtype=torch.float64, device=dev)
    r = torch.full((nobs,), 0.5, dtype=torch.float64, device=dev)
    out = torch.empty_like(x)
    plan = _native.Plan(ns, nobs, n, 0)
    ip = 0 if idx is None else idx.data_ptr()
    side = torch.cuda.Stream(dev)

    def call(s):
        assert lib.enkf_analysis_async_f64(plan.handle, x.data_ptr(), y.data_ptr(), ip, r.data_ptr(),
                                           out.data_ptr(), s) == 0

    with torch.cuda.stream(side):
        call(side.cuda_stream)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        call(torch.cuda.current_stream(dev).cuda_stream)
    s = torch.cuda.current_stream(dev)
    row = {}
    for mode in ("direct", "graph"):
        for _ in range(10):
            g.replay() if mode == "graph" else call(s.cuda_stream)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(s)
        for _ in range(reps):
            g.replay() if mode == "graph" else call(s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize(dev)
        row[mode + "_host_ms"] = (time.perf_counter() - t0) * 1e3 / reps
        row[mode + "_device_ms"] = a.elapsed_time(b) / reps
    res[name] = row
    del g, plan
print(json.dumps({"graph_probe": res, "reps": reps}))
