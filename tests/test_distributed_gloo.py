"""The multi-GPU orchestration (paper_1302_3876_b200.distributed) on CPU:
world_size 2 over gloo, with the device stages replaced by the numpy model of
the same three stages (tests/reduced_model.py).  Checks the row sharding, the
single Gram allreduce, the redundant level recursion and the cross-rank error
agreement; the CUDA stages themselves are covered by the -m gpu tests."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import reduced_model as M
from paper_1302_3876_b200 import _native
from paper_1302_3876_b200 import workloads as W
from paper_1302_3876_b200.distributed import ShardedAnalysis, obs_slice, shard_rows


class NumpyStages:
    """CPU stand-in for CudaStages (test infrastructure only)."""

    def __init__(self):
        self.code, self.msg = _native.ENKF_OK, "ok"
        self.level, self.den = 0, 0.0

    def partial_gram(self, x, y, idx, r):
        xo = x if idx is None else x[idx]
        if not (np.isfinite(xo).all() and np.isfinite(y).all()):
            self.code, self.msg = _native.ENKF_INVALID_ARGUMENT, "inputs contain non-finite entries"
        g = M.gram_analysis(xo, y, r) if len(r) else np.zeros((x.shape[1], 2 * x.shape[1]))
        return torch.from_numpy(np.ascontiguousarray(g))

    def levels(self, gram):
        try:
            a, _ = M.levels(gram.numpy())
        except M.ModelSingular as e:
            self.code, self.level, self.den = _native.ENKF_SINGULAR_UPDATE, e.level, e.denominator
            a = np.zeros((gram.shape[0], gram.shape[0]))
        return M.transform(a)

    def anomaly(self, x, t, out):
        out[...] = x @ t
        return out

    def status(self):
        return self.code, self.level, self.den, self.msg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, scenario, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = W.config4(10)
        ns = p.x.shape[0]
        lo, hi = shard_rows(ns, world, rank)
        a, b = obs_slice(p.indices, lo, hi)
        y = p.perturbed[a:b].copy()
        if scenario == "nan" and rank == 1:
            y[0, 0] = np.nan
        idx = p.indices[a:b] - lo
        x = p.x[lo:hi].copy()
        out = np.empty_like(x)
        runner = ShardedAnalysis(NumpyStages())
        try:
            runner.step(x, y, idx, p.r[a:b], out)
            q.put((rank, lo, hi, out, None))
        except Exception as e:  # noqa: BLE001
            q.put((rank, lo, hi, None, type(e).__name__))
    finally:
        dist.destroy_process_group()


def _run(world, scenario):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scenario, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    return sorted(res, key=lambda t: t[0])


def test_sharded_step_matches_unsharded_oracle():
    res = _run(2, "ok")
    p = W.config4(10)
    ref = oracle.analysis_step(p.x, p.perturbed, p.indices, p.r)
    xa = np.empty_like(p.x)
    for rank, lo, hi, out, err in res:
        assert err is None
        xa[lo:hi] = out
    assert np.abs(xa - ref).max() / np.abs(ref).max() <= 1e-12


def test_input_error_on_one_rank_raises_on_all():
    res = _run(2, "nan")
    assert [err for *_, err in res] == ["ValueError", "ValueError"]


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_shards_partition_observations(world):
    p = W.config4(10)
    ns = p.x.shape[0]
    seen = []
    for rank in range(world):
        lo, hi = shard_rows(ns, world, rank)
        a, b = obs_slice(p.indices, lo, hi)
        seen.extend(p.indices[a:b])
        assert np.all((p.indices[a:b] >= lo) & (p.indices[a:b] < hi))
    assert np.array_equal(np.asarray(seen), p.indices)
