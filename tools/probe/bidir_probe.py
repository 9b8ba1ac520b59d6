"""Bidirectional PCIe throughput with pinned buffers: one copy stream per direction
vs two (chunks alternate between the streams), 256 MiB chunks.

    python tools/probe/bidir_probe.py [GiB per direction, default 8]
"""
import json
import sys
import time

import torch

gib = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dev = torch.device("cuda", 0)
chunk = 256 << 20
n = (gib << 30) // chunk
h_in = torch.empty(gib << 30, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(gib << 30, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(gib << 30, dtype=torch.uint8, device=dev)
d_out = torch.empty(gib << 30, dtype=torch.uint8, device=dev)
h_in.fill_(1)
d_out.fill_(2)
res = {"gib_each_way": gib}
for k in (1, 2, 3):
    sin = [torch.cuda.Stream(dev) for _ in range(k)]
    sout = [torch.cuda.Stream(dev) for _ in range(k)]
    for rep in range(2):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for i in range(n):
            a, b = i * chunk, (i + 1) * chunk
            with torch.cuda.stream(sin[i % k]):
                d_in[a:b].copy_(h_in[a:b], non_blocking=True)
            with torch.cuda.stream(sout[i % k]):
                h_out[a:b].copy_(d_out[a:b], non_blocking=True)
        torch.cuda.synchronize(dev)
        el = time.perf_counter() - t0
    res[f"streams_{k}_gbs_each_way"] = (gib << 30) / el / 1e9
    # one direction only
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for i in range(n):
        a, b = i * chunk, (i + 1) * chunk
        with torch.cuda.stream(sin[i % k]):
            d_in[a:b].copy_(h_in[a:b], non_blocking=True)
    torch.cuda.synchronize(dev)
    res[f"streams_{k}_h2d_only_gbs"] = (gib << 30) / (time.perf_counter() - t0) / 1e9
print(json.dumps(res))
