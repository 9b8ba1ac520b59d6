"""Streamed host path probe: PCIe copy rates (H2D, D2H, both at once) with
pinned buffers, then the public API at config 5 with ENKF_HOST_TRACE=1 for a
few chunk sizes (phase times on stderr).

    python tools/probe/host_stream_probe.py [--log2-rows 26] [--chunks 64,256,1024]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def copy_rates(gb=16):
    dev = torch.device("cuda", 0)
    n = (gb << 30) // 8
    h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d_a = torch.empty(n, dtype=torch.float64, device=dev)
    d_b = torch.zeros(n, dtype=torch.float64, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name, fn in (("h2d", lambda: d_a.copy_(h_in, non_blocking=True)),
                     ("d2h", lambda: h_out.copy_(d_b, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter(); fn(); torch.cuda.synchronize()
        out[name + "_gbs"] = (gb << 30) / (time.perf_counter() - t) / 1e9
    torch.cuda.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    out["bidir_each_gbs"] = (gb << 30) / el / 1e9
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-rows", type=int, default=26)
    ap.add_argument("--chunks", default="64,256,1024")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    print(json.dumps(copy_rates()), flush=True)
    import paper_1302_3876_b200 as P
    from paper_1302_3876_b200 import _native
    from paper_1302_3876_b200 import workloads as W
    dev = torch.device("cuda", 0)
    cfg = 5
    scale = 26 - a.log2_rows
    d = W.device_problem_shard(cfg, 1, 0, dev, scale_log2=scale)
    x, y, idx, r = d["x"], d["perturbed"], d["idx"], d["r"]
    x_h = torch.empty(tuple(x.shape), dtype=torch.float64, pin_memory=True)
    y_h = torch.empty(tuple(y.shape), dtype=torch.float64, pin_memory=True)
    x_h.copy_(x)
    y_h.copy_(y)
    idx_h = idx.cpu().numpy()
    r_h = r.cpu().numpy()
    del x, y, d
    torch.cuda.empty_cache()
    h = P.SelectionOperator.from_indices(idx_h)
    obs = P.ObservationBatch(y=None, perturbed=y_h.numpy(), perturbations=None)
    for mb in [int(c) for c in a.chunks.split(",")]:
        os.environ["ENKF_HOST_TRACE"] = "1"
        os.environ["ENKF_HOST_CHUNK_MB"] = str(mb)
        _native._plans.clear()
        torch.cuda.empty_cache()
        P.analysis_step(x_h.numpy(), obs, h, r_h)
        ts = []
        for _ in range(a.reps):
            t = time.perf_counter()
            P.analysis_step(x_h.numpy(), obs, h, r_h)
            ts.append(time.perf_counter() - t)
        print(json.dumps({"chunk_mb": mb, "seconds": ts}), flush=True)


if __name__ == "__main__":
    main()
