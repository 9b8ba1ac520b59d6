"""A/B of the level-0 Gram: FP64 DMMA (gram128) vs the int8-digit tensor-core
path (ENKF_GRAM=i8), timed with CUDA events, results compared.

    python tools/probe/g8_ab.py [log2_obs] [log2_state] [reps] [modes, default fp64,i8]
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_1302_3876_b200 import _native  # noqa: E402

lg_o = int(sys.argv[1]) if len(sys.argv) > 1 else 20
lg_s = int(sys.argv[2]) if len(sys.argv) > 2 else lg_o + 3
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
modes = sys.argv[4].split(",") if len(sys.argv) > 4 else ["fp64", "i8"]
dev = torch.device("cuda", 0)
lib = _native.lib()
s = torch.cuda.current_stream().cuda_stream
n, ns, no = 128, 1 << lg_s, 1 << lg_o
g = torch.Generator(device=dev)
g.manual_seed(7)
x = torch.randn((ns, 1), dtype=torch.float64, device=dev, generator=g) + \
    (0.5 + 1.5 * torch.rand((ns, 1), dtype=torch.float64, device=dev, generator=g)) * \
    torch.randn((ns, n), dtype=torch.float64, device=dev, generator=g)
idx = torch.sort(torch.randperm(ns, device=dev, generator=g)[:no]).values
y = x[idx].mean(dim=1, keepdim=True) + torch.randn((no, n), dtype=torch.float64, device=dev, generator=g)
r = 0.25 + 0.75 * torch.rand((no,), dtype=torch.float64, device=dev, generator=g)
out = {"n_obs": no, "n_state": ns}
grams = {}
for mode in modes:
    os.environ["ENKF_GRAM"] = mode
    plan = _native.Plan(ns, no, n, 0)
    gram = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)
    ts = []
    for i in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        assert lib.enkf_plan_reset_status(plan.handle, s) == 0
        assert lib.enkf_ism_gram_f64(plan.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(),
                                     gram.data_ptr(), s) == 0
        b.record()
        torch.cuda.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
    st = _native.EnkfStatus()
    assert lib.enkf_plan_sync_status(plan.handle, s, ctypes.byref(st)) == 0, st.message
    grams[mode] = gram.clone()
    out[mode + "_ms"] = sorted(ts)
    del plan
for mode in modes[1:]:
    out[mode + "_max_rel_diff"] = (grams[mode] - grams[modes[0]]).abs().max().item() / grams[modes[0]].abs().max().item()
    out[mode + "_sym"] = (grams[mode][:, :n] - grams[mode][:, :n].T).abs().max().item()
print(json.dumps(out))
