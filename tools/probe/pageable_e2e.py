"""Config 5 through the public API with a caller's ordinary (pageable) numpy arrays:
analysis_step(x, obs, h, r) where x and the perturbed observations are plain
np.ndarray (the verdict's W9: the bench's e2e uses page-locked inputs).

    python tools/probe/pageable_e2e.py [scale_log2] [calls]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_1302_3876_b200 as P  # noqa: E402
from paper_1302_3876_b200 import workloads as W  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 0
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
d = W.device_problem_shard(5, 1, 0, dev, scale_log2=scale)
x = d["x"].cpu().numpy()            # pageable
y = d["perturbed"].cpu().numpy()    # pageable
r = d["r"].cpu().numpy()
idx = d["idx"].cpu().numpy()
del d
torch.cuda.empty_cache()
h = P.SelectionOperator.from_indices(idx)
obs = P.ObservationBatch(y=None, perturbed=y, perturbations=None)
times = []
for k in range(calls + 1):
    t0 = time.perf_counter()
    xa = P.analysis_step(x, obs, h, r)
    times.append(time.perf_counter() - t0)
    del xa
print(json.dumps({"n_state": x.shape[0], "n_obs": y.shape[0], "pageable_inputs": True,
                  "seconds_per_call": [round(t, 3) for t in times], "steps_per_s_warm": 1.0 / min(times[1:]),
                  "h2d_bytes": int(x.nbytes + y.nbytes + r.nbytes + idx.nbytes), "d2h_bytes": int(x.nbytes)}))
