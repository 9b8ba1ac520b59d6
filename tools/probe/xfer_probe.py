"""Host<->device transfer options for the e2e host path (one-off probe)."""
import ctypes, json, time
import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so.12") if False else None
out = {}
n = 1 << 29  # 4 GiB of doubles
d = torch.empty(n, dtype=torch.float64, device="cuda")
d.fill_(1.0)
torch.cuda.synchronize()
# pageable np.empty destination (fresh pages)
a = np.empty(n)
t = time.perf_counter(); torch.from_numpy(a).copy_(d); torch.cuda.synchronize(); out["d2h_pageable_fresh_gbs"] = n * 8 / (time.perf_counter() - t) / 1e9
t = time.perf_counter(); torch.from_numpy(a).copy_(d); torch.cuda.synchronize(); out["d2h_pageable_touched_gbs"] = n * 8 / (time.perf_counter() - t) / 1e9
t = time.perf_counter(); d.copy_(torch.from_numpy(a)); torch.cuda.synchronize(); out["h2d_pageable_gbs"] = n * 8 / (time.perf_counter() - t) / 1e9
b = np.empty(n)
t = time.perf_counter(); r = torch.cuda.cudart().cudaHostRegister(b.ctypes.data, b.nbytes, 0); out["host_register_fresh_s"] = time.perf_counter() - t; out["reg_rc"] = int(r)
t = time.perf_counter(); torch.from_numpy(b).copy_(d); torch.cuda.synchronize(); out["d2h_registered_gbs"] = n * 8 / (time.perf_counter() - t) / 1e9
t = time.perf_counter(); torch.cuda.cudart().cudaHostUnregister(b.ctypes.data); out["host_unregister_s"] = time.perf_counter() - t
t = time.perf_counter(); p = torch.empty(n, dtype=torch.float64, pin_memory=True); out["pinned_alloc_s"] = time.perf_counter() - t
t = time.perf_counter(); p.copy_(d); torch.cuda.synchronize(); out["d2h_pinned_gbs"] = n * 8 / (time.perf_counter() - t) / 1e9
t = time.perf_counter(); np.copyto(a, p.numpy()); out["host_memcpy_1thread_gbs"] = n * 8 / (time.perf_counter() - t) / 1e9
print(json.dumps(out))
