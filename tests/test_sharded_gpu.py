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


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_native_comm_world_one():
    """The product multi-GPU path (NCCL in the native layer: enkf_comm_init,
    enkf_plan_set_comm, one ncclAllReduce of [Gram | flags] inside the step) under a
    world-size-1 group: bitwise equal to the single-GPU step (the one-rank sum is a
    copy), the same on host buffers, input errors raise through the reduced flags,
    and the step replays from a captured CUDA graph."""
    import torch
    import torch.distributed as dist
    from paper_1302_3876_b200.distributed import NativeComm, NativeShardedAnalysis
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    try:
        p = W.config4(8)
        ns, nobs, n = p.shape
        comm = NativeComm(dev)
        runner = NativeShardedAnalysis(ns, nobs, n, dev, comm)
        x = torch.from_numpy(p.x).to(dev)
        y = torch.from_numpy(p.perturbed).to(dev)
        idx = torch.from_numpy(p.indices).to(dev)
        r = torch.from_numpy(p.r).to(dev)
        out = runner.step(x, y, idx, r, torch.empty_like(x))
        assert np.array_equal(out.cpu().numpy(), _unsharded(p, dev))
        out_h = np.empty_like(p.x)
        runner.step_host(p.x, p.perturbed, p.indices, p.r, out_h)
        assert np.array_equal(out_h, out.cpu().numpy())
        bad = r.clone()
        bad[3] = -1.0
        with pytest.raises(ValueError):
            runner.step(x, y, idx, bad, torch.empty_like(x))
        big = idx.clone()
        big[-1] = ns
        with pytest.raises(IndexError):
            runner.step(x, y, big, r, torch.empty_like(x))
        # graph capture of the async sharded step (collective included)
        g_out = torch.empty_like(x)
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            runner.step(x, y, idx, r, g_out, check=False)  # warm-up on the capture stream
        torch.cuda.current_stream(dev).wait_stream(s)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            runner.step(x, y, idx, r, g_out, check=False)
        g_out.zero_()
        graph.replay()
        torch.cuda.synchronize(dev)
        runner.raise_for_status()
        assert torch.equal(g_out, out)
        del graph, runner
        comm.close()
    finally:
        dist.destroy_process_group()


def _two_rank_worker(rank, world, port, path, bad_rank):
    import torch
    import torch.distributed as dist
    from paper_1302_3876_b200.distributed import NativeComm, NativeShardedAnalysis
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=dev)
    try:
        p = W.config4(8)
        ns, nobs, n = p.shape
        lo, hi = shard_rows(ns, world, rank)
        a, b = obs_slice(p.indices, lo, hi)
        comm = NativeComm(dev)
        runner = NativeShardedAnalysis(hi - lo, b - a, n, dev, comm)
        x = torch.from_numpy(p.x[lo:hi]).to(dev)
        y = torch.from_numpy(p.perturbed[a:b]).to(dev)
        r = torch.from_numpy(p.r[a:b]).to(dev)
        idx = torch.from_numpy(p.indices[a:b] - lo).to(dev)
        out = runner.step(x, y, idx, r, torch.empty_like(x))
        np.save(f"{path}.{rank}.npy", out.cpu().numpy())
        if rank == bad_rank:
            r[0] = float("nan")
        try:
            runner.step(x, y, idx, r, torch.empty_like(x))
            raised = "none"
        except ValueError:
            raised = "ValueError"
        open(f"{path}.{rank}.err", "w").write(raised)
        del runner
        comm.close()
    finally:
        dist.destroy_process_group()


def test_native_comm_two_ranks(tmp_path):
    """Two ranks on two GPUs (skipped below 2 GPUs): the sharded step with the
    native NCCL exchange equals the unsharded step to reduction-order rounding, and
    a bad input on one rank raises ValueError on both."""
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    world = 2
    path = str(tmp_path / "xa")
    mp.spawn(_two_rank_worker, args=(world, _free_port(), path, 1), nprocs=world, join=True)
    p = W.config4(8)
    out = np.empty_like(p.x)
    for rank in range(world):
        lo, hi = shard_rows(p.x.shape[0], world, rank)
        out[lo:hi] = np.load(f"{path}.{rank}.npy")
        assert open(f"{path}.{rank}.err").read() == "ValueError", rank
    dev = torch.device("cuda", 0)
    assert rel_err(out, _unsharded(p, dev)) <= 1e-12
