"""The multi-GPU decomposition on one GPU, without ranks that wait on each other:
G row shards are run one after another with the product stages (CudaStages,
libenkf_b200.so), their partial Grams are summed in fixed order (what the NCCL
allreduce does), and every shard is updated with the shared T.  The result must
equal the unsharded step (SURVEY §4 "G-count independence": only the reduction
order differs), and ShardedAnalysis itself runs under a world-size-1 NCCL group.
"""

import os
import socket

import numpy as np
import pytest

import oracle
from golden_io import rel_err
import paper_1302_3876_b200 as P
from paper_1302_3876_b200 import workloads as W
from paper_1302_3876_b200.distributed import CudaStages, ShardedAnalysis, obs_slice, shard_rows

pytestmark = pytest.mark.gpu


def _unsharded(p, dev):
    import torch
    h = P.SelectionOperator.from_indices(p.indices)
    obs = P.ObservationBatch(y=None, perturbed=torch.from_numpy(p.perturbed).to(dev), perturbations=None)
    return P.analysis_step(torch.from_numpy(p.x).to(dev), obs, h, torch.from_numpy(p.r).to(dev)).cpu().numpy()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sequential_shards_equal_unsharded(world):
    import torch
    dev = torch.device("cuda", 0)
    p = W.config4(8)
    ns, nobs, n = p.shape
    full = _unsharded(p, dev)
    parts, shards = [], []
    for rank in range(world):
        lo, hi = shard_rows(ns, world, rank)
        a, b = obs_slice(p.indices, lo, hi)
        st = CudaStages(hi - lo, max(b - a, 1), n, dev)
        x = torch.from_numpy(p.x[lo:hi]).to(dev)
        y = torch.from_numpy(p.perturbed[a:b]).to(dev)
        r = torch.from_numpy(p.r[a:b]).to(dev)
        idx = torch.from_numpy(p.indices[a:b] - lo).to(dev)
        parts.append(st.partial_gram(x, y, idx, r).clone())
        shards.append((st, x, lo, hi))
    gram = parts[0].clone()
    for g in parts[1:]:
        gram += g  # the allreduce, in rank order
    out = np.empty_like(p.x)
    for st, x, lo, hi in shards:
        t = st.levels(gram.clone())
        xa = torch.empty_like(x)
        st.anomaly(x, t, xa)
        torch.cuda.synchronize()
        assert st.status()[0] == 0
        out[lo:hi] = xa.cpu().numpy()
    assert rel_err(out, full) <= 1e-12
    assert rel_err(out, oracle.analysis_step_chunked(p.x, p.perturbed, p.indices, p.r)) <= 1e-9


def test_sharded_analysis_world_one_nccl():
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        p = W.config4(8)
        ns, nobs, n = p.shape
        runner = ShardedAnalysis(CudaStages(ns, nobs, n, dev))
        x = torch.from_numpy(p.x).to(dev)
        out = runner.step(x, torch.from_numpy(p.perturbed).to(dev), torch.from_numpy(p.indices).to(dev),
                          torch.from_numpy(p.r).to(dev), torch.empty_like(x))
        assert rel_err(out.cpu().numpy(), _unsharded(p, dev)) <= 1e-13
        bad = torch.from_numpy(p.r).to(dev).clone()
        bad[3] = -1.0
        with pytest.raises(ValueError):
            runner.step(x, torch.from_numpy(p.perturbed).to(dev), torch.from_numpy(p.indices).to(dev), bad,
                        torch.empty_like(x))
    finally:
        dist.destroy_process_group()
