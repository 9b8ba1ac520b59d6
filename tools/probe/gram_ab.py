"""A/B of the Gram forms at config 5 (or 2^-s of it): the Gram alone and the whole
step, per ENKF_GRAM mode, alternating, CUDA events; Grams compared bitwise.

    python tools/probe/gram_ab.py [scale_log2] [modes, e.g. i8ls,fp64] [reps]
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_1302_3876_b200 import _native  # noqa: E402
from paper_1302_3876_b200 import workloads as W  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 0
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["i8ls", "fp64"]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dev = torch.device("cuda", 0)
lib = _native.lib()
s = torch.cuda.current_stream().cuda_stream
d = W.device_problem_shard(5, 1, 0, dev, scale_log2=scale)
x, y, idx, r = d["x"], d["perturbed"], d["idx"], d["r"]
ns, no, n = x.shape[0], y.shape[0], x.shape[1]
xa = torch.empty_like(x)
plans = {}
for m in modes:
    os.environ["ENKF_GRAM"] = m
    plans[m] = _native.Plan(ns, no, n, 0)
os.environ.pop("ENKF_GRAM", None)
gram = {m: torch.empty((n, 2 * n), dtype=torch.float64, device=dev) for m in modes}
res = {m: {"gram_ms": [], "step_ms": []} for m in modes}


def ev_time(fn, k=1):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


for rep in range(reps):
    for m in modes:
        h = plans[m].handle
        lib.enkf_plan_reset_status(h, s)
        res[m]["gram_ms"].append(ev_time(lambda: lib.enkf_ism_gram_f64(h, x.data_ptr(), y.data_ptr(), idx.data_ptr(),
                                                                      r.data_ptr(), gram[m].data_ptr(), s)))
        st = _native.EnkfStatus()
        assert lib.enkf_plan_sync_status(h, s, ctypes.byref(st)) == 0, (m, st.message)
        res[m]["step_ms"].append(ev_time(lambda: lib.enkf_analysis_async_f64(
            h, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(), xa.data_ptr(), s), k=3))
        assert lib.enkf_plan_sync_status(h, s, ctypes.byref(st)) == 0, (m, st.message)
out = {"scale_log2": scale, "n_obs": no, "n_state": ns}
for m in modes:
    g = res[m]
    out[m] = {"gram_ms_med": float(np.median(g["gram_ms"][1:] or g["gram_ms"])),
              "step_ms_med": float(np.median(g["step_ms"][1:] or g["step_ms"])),
              "gram_ms": [round(v, 3) for v in g["gram_ms"]], "step_ms": [round(v, 3) for v in g["step_ms"]]}
if len(modes) > 1:
    a = gram[modes[0]].cpu().numpy()
    for m in modes[1:]:
        b = gram[m].cpu().numpy()
        out[f"gram_{m}_vs_{modes[0]}"] = {"bitwise_equal": bool(np.array_equal(a, b)),
                                          "max_rel": float(np.abs(a - b).max() / np.abs(a).max())}
print(json.dumps(out))
