"""Host memcpy bandwidth (pageable -> pinned) with 1..16 threads, and the
pageable host-API call at config 4 split into its parts."""
import json, os, sys, time, threading
import numpy as np
import torch
sys.path.insert(0, os.getcwd())

n = (4 << 30) // 8
src = np.random.default_rng(1).standard_normal(n)
dst = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
out = {"cpus": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
for nt in (1, 4, 8, 16, 32):
    per = n // nt
    def work(t):
        np.copyto(dst[t * per:(t + 1) * per], src[t * per:(t + 1) * per])
    t0 = time.perf_counter()
    th = [threading.Thread(target=work, args=(t,)) for t in range(nt)]
    [x.start() for x in th]; [x.join() for x in th]
    out[f"memcpy_{nt}t_gbs"] = n * 8 / (time.perf_counter() - t0) / 1e9
print(json.dumps(out), flush=True)
import paper_1302_3876_b200 as P
from paper_1302_3876_b200 import workloads as W
p = W.config4(0)
h = P.SelectionOperator.from_indices(p.indices)
obs = P.ObservationBatch(y=None, perturbed=p.perturbed, perturbations=None)
P.analysis_step(p.x, obs, h, p.r)
for _ in range(2):
    t0 = time.perf_counter(); P.analysis_step(p.x, obs, h, p.r); print("pageable host call s", time.perf_counter() - t0, flush=True)
