#!/bin/bash
# Gram pass times (library events) per library variant: gram_pass_ab.sh ROUNDS VAR...
# ("-" = product build; "KEY=VALUE" = product build with that environment variable)
R=${1:-2}; shift
for i in $(seq $R); do for v in "$@"; do vv=$v; [ "$v" = "-" ] && vv=""; ee="ENKF_UNUSED=1"; case "$v" in *=*) ee="$v"; vv="";; esac
env "$ee" ENKF_LIB_VARIANT=$vv ENKF_AB_LABEL="$v" python - <<'PY'
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1302_3876_b200 import _native
from paper_1302_3876_b200 import workloads as W
dev = torch.device("cuda", 0); lib = _native.lib(); s = torch.cuda.current_stream().cuda_stream
lib.enkf_debug_set_gram_events.argtypes = [ctypes.c_void_p, ctypes.c_int32]
lib.enkf_debug_gram_times.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]
d = W.device_problem_shard(5, 1, 0, dev, scale_log2=0)
x, y, idx, r = d["x"], d["perturbed"], d["idx"], d["r"]
ns, no, n = x.shape[0], y.shape[0], x.shape[1]
plan = _native.Plan(ns, no, n, 0); gram = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)
h = plan.handle; sl, mm = [], []
for k in range(6):
    lib.enkf_debug_set_gram_events(h, 1)
    lib.enkf_ism_gram_f64(h, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(), gram.data_ptr(), s)
    torch.cuda.synchronize(); two = (ctypes.c_float * 2)(); lib.enkf_debug_gram_times(h, two)
    sl.append(round(two[0], 3)); mm.append(round(two[1], 3))
g = gram.cpu().numpy()
os.environ["ENKF_GRAM"] = "fp64"; p64 = _native.Plan(ns, no, n, 0); g64 = torch.empty_like(gram)
lib.enkf_ism_gram_f64(p64.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(), g64.data_ptr(), s); torch.cuda.synchronize()
a = g64.cpu().numpy()
print("variant=%s" % os.environ.get("ENKF_AB_LABEL", ""), "slice", sl, "mma", mm, "vs_fp64", float(np.abs(a - g).max() / np.abs(a).max()), "sym", float(np.abs(g[:, :n] - g[:, :n].T).max()))
PY
done; done
