"""Row-sharded analysis step across the GPUs of one node (one rank per GPU).

Partitioning: rank g owns the contiguous state rows
[g Ns/G, (g+1) Ns/G) and the observation rows whose sorted index falls in
that range (contiguous because H's indices are strictly increasing,
enkf.py:41-42).  Everything is row-local except the level-0 Gram
[V'R^-1 V | V'R^-1 D] (N x 2N): each rank computes its partial over its own
observation rows, ONE allreduce (sum) over torch.distributed — NCCL over
NVLink on the box — makes it global, and every rank then runs the N
Sherman-Morrison levels on the identical reduced Gram (no broadcast) and
updates its own state rows.  Per step that is a single 2 N^2 fp64 allreduce
(256 KiB at N = 128) instead of the reference's per-level column exchange.

Two forms:

* `NativeShardedAnalysis` (the product path, bench.py's N > 1 leg): the exchange
  lives in the native layer.  `NativeComm` creates an NCCL communicator inside
  libenkf_b200.so (the 128-byte unique id is handed out over torch.distributed),
  the shard's plan gets it attached, and one C call per step runs the local Gram,
  the ncclAllReduce of [Gram | input-check flags] on the compute stream, the
  levels and the local anomaly update — every rank returns the same status, with
  no extra collective or host synchronisation (include/enkf_b200.h).
* `ShardedAnalysis` over pluggable stages: the same orchestration in Python with
  `torch.distributed.all_reduce`, kept so the sharding logic can be exercised on
  CPU with the gloo backend (tests/test_distributed_gloo.py).  Its product stages
  are `CudaStages` (libenkf_b200.so); nothing here falls back to the CPU.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import SingularUpdateError


def shard_rows(n_state: int, world: int, rank: int):
    """Contiguous state-row shard [lo, hi) of `rank`."""
    base, extra = divmod(n_state, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (rank < extra)


def obs_slice(indices, lo: int, hi: int):
    """Observation rows [a, b) whose state index lies in [lo, hi) (None = identity)."""
    if indices is None:
        return lo, hi
    a = int(np.searchsorted(indices, lo, side="left"))
    b = int(np.searchsorted(indices, hi, side="left"))
    return a, b


class CudaStages:
    """The three device stages of one rank, on libenkf_b200.so."""

    def __init__(self, n_state_local: int, n_obs_local: int, n_ens: int, device):
        import torch

        self.torch = torch
        self.device = device
        self.n = n_ens
        self.plan = _native.Plan(n_state_local, n_obs_local, n_ens, device.index)
        self.lib = _native.lib()
        self.gram = torch.empty((n_ens, 2 * n_ens), dtype=torch.float64, device=device)
        self.a = torch.empty((n_ens, n_ens), dtype=torch.float64, device=device)
        self.t = torch.empty((n_ens, n_ens), dtype=torch.float64, device=device)
        self.den = torch.empty(n_ens, dtype=torch.float64, device=device)

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def new_gram(self):
        return self.gram

    def partial_gram(self, x, y, idx, r):
        s = self._stream()
        self.lib.enkf_plan_reset_status(self.plan.handle, s)
        rc = self.lib.enkf_ism_gram_f64(self.plan.handle, x.data_ptr(), y.data_ptr(),
                                        0 if idx is None else idx.data_ptr(), r.data_ptr(),
                                        self.gram.data_ptr(), s)
        _native.raise_for_status(rc, None, "enkf_ism_gram_f64")
        return self.gram

    def levels(self, gram):
        rc = self.lib.enkf_ism_levels_f64(self.plan.handle, gram.data_ptr(), self.a.data_ptr(),
                                          self.t.data_ptr(), self.den.data_ptr(), self._stream())
        _native.raise_for_status(rc, None, "enkf_ism_levels_f64")
        return self.t

    def anomaly(self, x, t, out):
        rc = self.lib.enkf_anomaly_update_f64(self.plan.handle, x.data_ptr(), t.data_ptr(),
                                              out.data_ptr(), x.shape[0], self._stream())
        _native.raise_for_status(rc, None, "enkf_anomaly_update_f64")
        return out

    def status(self):
        """(code, level, denominator, message) after draining the stream."""
        st = _native.EnkfStatus()
        code = self.lib.enkf_plan_sync_status(self.plan.handle, self._stream(), ctypes.byref(st))
        return code, st.level, st.denominator, st.message.decode(errors="replace")


class ShardedAnalysis:
    """One analysis step over all ranks of `group` (default: the world).

    `step(x, y, idx, r, out)` takes this rank's shard: x = X[lo:hi] (rows,
    N), y / r = the perturbed observations / variances of its observation rows,
    idx = their state indices relative to lo (None for the identity), and
    writes X^A[lo:hi] into `out` (may be `x`).
    """

    def __init__(self, stages, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.stages = stages
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def step(self, x, y, idx, r, out, check: bool = True, events=None):
        """`events` (bench only): 5 CUDA events recorded at the stage
        boundaries (gram | allreduce | levels | anomaly)."""
        rec = (lambda i: events[i].record()) if events is not None else (lambda i: None)
        rec(0)
        gram = self.stages.partial_gram(x, y, idx, r)
        rec(1)
        if self.world > 1:
            self.dist.all_reduce(gram, group=self.group)
        rec(2)
        t = self.stages.levels(gram)
        rec(3)
        self.stages.anomaly(x, t, out)
        rec(4)
        if check:
            self.raise_for_status()
        return out

    def raise_for_status(self):
        """Agree on the outcome across ranks (a local input error on one rank
        raises on every rank) and raise the reference's exception type."""
        code, level, den, msg = self.stages.status()
        if self.world > 1:
            import torch

            dev = getattr(self.stages, "device", None)
            if dev is None or self.dist.get_backend(self.group) == "gloo":
                dev = torch.device("cpu")
            flag = torch.tensor([code], dtype=torch.int64, device=dev)
            self.dist.all_reduce(flag, op=self.dist.ReduceOp.MAX, group=self.group)
            gcode = int(flag.item())
            if gcode != code:
                code, msg = gcode, f"raised on another rank (code {gcode})"
        if code == _native.ENKF_SINGULAR_UPDATE:
            raise SingularUpdateError(int(level), float(den))
        if code != _native.ENKF_OK:
            st = _native.EnkfStatus()
            st.code = code
            st.message = msg.encode()[:255]
            _native.raise_for_status(code, st, "sharded analysis step")


class NativeComm:
    """An NCCL communicator created by libenkf_b200.so (ncclCommInitRank) for the
    ranks of `group` (default: the world), one per GPU.  Rank 0 draws the unique id
    (ncclGetUniqueId); it reaches the other ranks through a torch.distributed
    broadcast (any backend)."""

    def __init__(self, device, group=None):
        import torch
        import torch.distributed as dist

        self.device = device
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        lib = _native.lib()
        st = _native.EnkfStatus()
        uid = (ctypes.c_ubyte * 128)()
        if self.rank == 0:
            _native.raise_for_status(lib.enkf_comm_unique_id(uid, ctypes.byref(st)), st, "enkf_comm_unique_id")
        if self.world > 1:
            on_cuda = dist.get_backend(group) == "nccl"
            buf = torch.tensor(list(bytes(uid)), dtype=torch.uint8,
                               device=device if on_cuda else torch.device("cpu"))
            dist.broadcast(buf, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
            uid = (ctypes.c_ubyte * 128)(*buf.cpu().tolist())
        self._h = ctypes.c_void_p()
        code = lib.enkf_comm_init(uid, self.world, self.rank, device.index, ctypes.byref(self._h), ctypes.byref(st))
        _native.raise_for_status(code, st, "enkf_comm_init")

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h is not None and self._h.value and _native._lib is not None:
            _native._lib.enkf_comm_destroy(self._h)
        self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NativeShardedAnalysis:
    """One rank's shard of the analysis step with the exchange in the native layer
    (see the module docstring).  `step(x, y, idx, r, out)` takes CUDA tensors:
    x = X[lo:hi] (rows, N), y / r = this shard's perturbed observations /
    variances, idx = their state indices relative to lo (None for the identity),
    and writes X^A[lo:hi] into `out` (may be `x`).  With check=True it reads the
    status (one device->host copy) and raises the reference's exception type —
    the same on every rank."""

    def __init__(self, n_state_local: int, n_obs_local: int, n_ens: int, device, comm: NativeComm):
        import torch

        self.torch = torch
        self.device = device
        self.comm = comm
        self.plan = _native.Plan(n_state_local, n_obs_local, n_ens, device.index)
        self.lib = _native.lib()
        st = _native.EnkfStatus()
        _native.raise_for_status(self.lib.enkf_plan_set_comm(self.plan.handle, comm.handle, ctypes.byref(st)),
                                 st, "enkf_plan_set_comm")

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def step(self, x, y, idx, r, out, check: bool = True):
        code = self.lib.enkf_analysis_async_f64(self.plan.handle, x.data_ptr(), y.data_ptr(),
                                                0 if idx is None else idx.data_ptr(), r.data_ptr(),
                                                out.data_ptr(), self._stream())
        if code != _native.ENKF_OK:
            # a failed launch (e.g. the collective): read the plan's status for the message
            st = _native.EnkfStatus()
            self.lib.enkf_plan_sync_status(self.plan.handle, self._stream(), ctypes.byref(st))
            _native.raise_for_status(code, st, "enkf_analysis_async_f64 (sharded)")
        if check:
            self.raise_for_status()
        return out

    def step_host(self, x_h, y_h, idx_h, r_h, out_h):
        """The same shard step on host (numpy) buffers through enkf_analysis_host_f64:
        copies in, the step with the NCCL exchange, X^A out."""
        import numpy as np

        st = _native.EnkfStatus()
        idx_c = None if idx_h is None else np.ascontiguousarray(idx_h, dtype=np.int64)  # held across the call
        ptr = lambda a: a.ctypes.data if a is not None else None  # noqa: E731
        code = self.lib.enkf_analysis_host_f64(self.plan.handle, ptr(x_h), ptr(y_h), ptr(idx_c),
                                               ptr(r_h), ptr(out_h), ctypes.byref(st))
        _native.raise_for_status(code, st, "enkf_analysis_host_f64 (sharded)")
        return out_h

    def raise_for_status(self):
        st = _native.EnkfStatus()
        code = self.lib.enkf_plan_sync_status(self.plan.handle, self._stream(), ctypes.byref(st))
        _native.raise_for_status(code, st, "sharded analysis step")
