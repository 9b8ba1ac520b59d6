"""Per-shard partial Gram, int8 vs FP64 (debug aid for the sharded decomposition)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_1302_3876_b200 import workloads as W  # noqa: E402
from paper_1302_3876_b200.distributed import CudaStages, obs_slice, shard_rows  # noqa: E402

dev = torch.device("cuda", 0)
p = W.config4(8)
ns, nobs, n = p.shape
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for rank in range(world):
    lo, hi = shard_rows(ns, world, rank)
    a, b = obs_slice(p.indices, lo, hi)
    res = {}
    for mode in ("fp64", "i8"):
        os.environ["ENKF_GRAM"] = mode
        st = CudaStages(hi - lo, max(b - a, 1), n, dev)
        x = torch.from_numpy(p.x[lo:hi]).to(dev)
        y = torch.from_numpy(p.perturbed[a:b]).to(dev)
        r = torch.from_numpy(p.r[a:b]).to(dev)
        idx = torch.from_numpy(p.indices[a:b] - lo).to(dev)
        res[mode] = st.partial_gram(x, y, idx, r).clone().cpu().numpy()
        torch.cuda.synchronize()
    d = np.abs(res["i8"] - res["fp64"])
    print(rank, b - a, d.max() / np.abs(res["fp64"]).max(), np.unravel_index(d.argmax(), d.shape), flush=True)

if len(sys.argv) > 2:
    rank = int(sys.argv[2])
    lo, hi = shard_rows(ns, world, rank)
    a, b = obs_slice(p.indices, lo, hi)
    xs = p.x[lo:hi]
    xo = xs[p.indices[a:b] - lo]
    y = p.perturbed[a:b]
    r = p.r[a:b]
    sr = np.sqrt(1.0 / r)
    P = sr[:, None] * (xo - xo.mean(axis=1, keepdims=True))
    Q = sr[:, None] * (y - xo)
    samp = np.arange(0, b - a, 16)
    for name, M in (("P", P), ("Q", Q)):
        full = np.abs(M).max(axis=0)
        sm = np.abs(M[samp]).max(axis=0)
        ratio = full / sm
        print(name, "max full/sampled ratio", ratio.max(), "col", ratio.argmax(), flush=True)
    os.environ["ENKF_GRAM"] = "i8"
    st = CudaStages(hi - lo, max(b - a, 1), n, dev)
    g = st.partial_gram(torch.from_numpy(xs).to(dev), torch.from_numpy(y).to(dev),
                        torch.from_numpy(p.indices[a:b] - lo).to(dev), torch.from_numpy(r).to(dev)).cpu().numpy()
    ref = np.concatenate([P.T @ P / (n - 1), P.T @ Q / np.sqrt(n - 1)], axis=1)
    d = np.abs(g - ref) / np.abs(ref).max()
    bad = np.argwhere(d > 1e-10)
    print("bad entries", len(bad), bad[:20].tolist(), flush=True)
