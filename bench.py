"""Benchmark of the B200 EnKF analysis step (iterative Sherman-Morrison).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--impl ours|reference]

N > 1: run under torchrun (one rank per GPU; the driver's launch), or plain
`python bench.py --gpus N`, which re-launches itself under torchrun with N ranks
(and exits non-zero if fewer than N GPUs are visible).  One JSON line on rank 0.

A "step" = one full analysis step (BASELINE.json metric "EnKF analysis
steps/sec") through the product entry point enkf_analysis_async_f64: level-0
Gram pass over the observed rows, (N > 1) ONE ncclAllReduce of the N x 2N Gram
with the input-check flags appended, issued by the native layer on the compute
stream, the N Sherman-Morrison levels, and the anomaly update X^A = X T over
every state row.  Workload = config 5 (n_state = 2^26, n_ens = 128,
n_obs = 2^23) by default: the config BASELINE.json's 1/2/4/8-GPU scaling is
quoted on; it fits one B200 (X + X^A + Y + the Gram's operand images = 148 GB).
State rows (and the observation rows they own) are sharded across ranks:
strong scaling, the problem is fixed.

  value : steps/s, whole job, inputs resident in HBM, CUDA-event timed on the
          launching stream, barrier + synchronize around the K steps, max over
          ranks.  The default arithmetic is fp64 EMULATED on the int8 tensor
          cores (exact byte-digit products, one rounding; `dtype` says so);
          `strict_fp64` times the all-IEEE-FP64 DMMA path in the same run.
  e2e   : the same metric through the public API with host buffers, host->device
          and device->host copies inside the timed region (N = 1:
          `analysis_step(numpy)`; N > 1: each rank's shard through
          enkf_analysis_host_f64 with the communicator attached).
  roofline : the anomaly-update kernel (the dominant one): HBM GB/s of X read +
          X^A written against MEASURED_PEAKS.json; `roofline_step` = the step's
          compulsory bytes / step time; `ism_sweep` = the Gram's HBM-streaming
          pass on compulsory bytes, with the DRAM-traffic ratio from ncu.
  cpu_baseline : the CPU oracle (oracle/, a numpy/OpenBLAS restatement of the
          reference, which is pure Python) on two bounded row samples of the same
          workload (linearity shown), extrapolated linearly to the full size.
"""

from __future__ import annotations

import argparse
import glob
import json
import os
import socket
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_DMMA_PEAK_TFLOPS = 37.07  # measured: profiles/r01_fp64_probe.json (DMMA m8n8k4, 148 SMs)
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
EMULATED_DTYPE = "f64 (int8-digit emulation on tcgen05: exact byte-digit products, 26 digit pairs, one rounding)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--scale-log2", type=int, default=0, help="shrink n_state/n_obs by 2^s (testing)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the strict-FP64 leg, the stage/pass breakdown and the overflow-cliff probe")
    ap.add_argument("--cpu-sample-log2", type=int, default=None)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_name(cfg, s):
    from paper_1302_3876_b200 import workloads as W
    z = W.SIZES[cfg]
    if cfg <= 3:
        return f"config{cfg}: n_state={z['ns']} n_ens={z['nens']} n_obs={z['nobs']}"
    return (f"config{cfg}: n_state=2^{(z['ns'] >> s).bit_length() - 1} n_ens={z['nens']} "
            f"n_obs=2^{(z['nobs'] >> s).bit_length() - 1}")


def hbm_peak():
    try:
        peaks = json.load(open(PEAKS_PATH))
        return float(peaks["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- self-launch (N > 1)
def self_launch(args):
    """`python bench.py --gpus N` outside torchrun: re-run under torchrun with N
    ranks on 127.0.0.1, NCCL communicator-init lines logged (NCCL_DEBUG=INFO,
    SUBSYS=INIT) to per-rank files that rank 0 folds into its JSON line."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but only {have} CUDA device(s) are visible"}),
              file=sys.stderr, flush=True)
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd, env=dict(os.environ)))


def nccl_log_setup():
    """Per-rank NCCL init logs (unless the caller configured NCCL_DEBUG itself)."""
    if "NCCL_DEBUG" in os.environ:
        return None
    run = os.environ.get("TORCHELASTIC_RUN_ID", "") + os.environ.get("MASTER_PORT", "")
    d = os.path.join(tempfile.gettempdir(), f"enkf_nccl_{run}")
    os.makedirs(d, exist_ok=True)
    os.environ["NCCL_DEBUG"] = "INFO"
    os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
    os.environ["NCCL_DEBUG_FILE"] = os.path.join(d, "nccl.%h.%p.log")
    return d


def nccl_init_lines(d):
    if not d:
        return None
    keep = []
    for f in sorted(glob.glob(os.path.join(d, "nccl.*.log"))):
        for line in open(f, errors="replace"):
            if "Init COMPLETE" in line or "ncclCommInitRank comm" in line:
                keep.append(line.strip())
    return keep[:32]


# ----------------------------------------------------------------------------- CPU legs
def cpu_sample_log2(cfg: int, scale: int) -> int:
    """The smaller of the two CPU samples (the larger is 4x its rows): config 5 at
    1/64 and 1/16 (the 1/256 sample is dominated by per-level Python overhead: 4x the
    rows took only 2.3x the time on the box), config 4 at 1/16 and 1/4."""
    return {4: 4, 5: 6}[cfg] - scale if cfg in (4, 5) else 0


def _threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count()


def run_cpu_oracle(cfg, scale, sample_log2, steps, warmup):
    """Time the oracle port (numpy + OpenBLAS, all host threads).  Configs 1-3: the
    full configuration.  Configs 4/5: two row samples 1/2^s and 1/2^(s-2) (the
    step is linear in n_state and n_obs at fixed n_ens; the per-row cost of the two
    shows it), value extrapolated from the larger sample."""
    import oracle
    from paper_1302_3876_b200 import workloads as W

    def timed(p, k):
        for _ in range(warmup):
            oracle.analysis_step_chunked(p.x, p.perturbed, p.indices, p.r)
        times = []
        for _ in range(max(1, k)):
            t0 = time.perf_counter()
            oracle.analysis_step_chunked(p.x, p.perturbed, p.indices, p.r)
            times.append(time.perf_counter() - t0)
        return min(times), len(times)

    if cfg <= 3:
        p = small_problem(cfg)
        t, k = timed(p, max(3, steps))
        return dict(value=1.0 / t, unit="steps/s", cores=int(_threads()), kind="port", extrapolated=False,
                    sample=f"oracle/ (numpy+OpenBLAS restatement of enkf.analysis_step) on the full {p.name} "
                           f"{p.shape}, best of {k}: {t * 1e3:.3f} ms", sample_seconds=t)
    mk = W.config4 if cfg == 4 else W.config5
    s_small = max(0, sample_log2)
    s_big = max(0, s_small - 2)
    out = {}
    for s in (s_small, s_big):
        p = mk(scale + s)
        t, k = timed(p, steps if s == s_big else 1)
        out[s] = (t, k, p.shape)
        del p
    t_b, k_b, shp = out[s_big]
    t_s = out[s_small][0]
    factor = 2 ** s_big
    return dict(value=1.0 / (t_b * factor), unit="steps/s", cores=int(_threads()), kind="port", extrapolated=True,
                sample=(f"oracle/ (numpy+OpenBLAS restatement of enkf.analysis_step) on a 1/{factor} row sample "
                        f"(n_state={shp[0]}, n_obs={shp[1]}, n_ens={shp[2]}), best of {k_b}: {t_b:.3f} s; "
                        f"value = 1/({t_b:.3f} s x {factor}); the 1/{2 ** s_small} sample took {t_s:.3f} s"),
                sample_seconds=t_b,
                linearity={"samples": [f"1/{2 ** s_small}", f"1/{factor}"], "seconds": [t_s, t_b],
                           "time_ratio_for_4x_rows": t_b / t_s})


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        import statistics
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        sm = [v for v in (num(r[1]) for r in self.rows) if v is not None]
        mx = [v for v in (num(r[2]) for r in self.rows) if v is not None]
        pw = [v for v in (num(r[3]) for r in self.rows if len(r) > 3) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w": statistics.median(pw) if pw else None}


class EnergyMeter:
    """Board energy over a region from NVML's cumulative counter
    (nvmlDeviceGetTotalEnergyConsumption, mJ); None where unavailable."""

    def __init__(self, index):
        self.index = index
        self.joules = None
        self._h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self._h = None

    def _read(self):
        try:
            return float(self._nv.nvmlDeviceGetTotalEnergyConsumption(self._h)) / 1e3
        except Exception:
            return None

    def __enter__(self):
        self._e0 = self._read() if self._h is not None else None
        return self

    def __exit__(self, *a):
        if self._e0 is not None:
            e1 = self._read()
            self.joules = (e1 - self._e0) if e1 is not None else None


# ----------------------------------------------------------------------------- GPU leg
class Runner:
    """One rank's analysis step through the product entry point
    enkf_analysis_async_f64 (communicator attached when N > 1)."""

    def __init__(self, ns_loc, nobs_loc, n, dev, comm, env=None):
        import ctypes

        from paper_1302_3876_b200 import _native
        self.ctypes = ctypes
        self.native = _native
        self.lib = _native.lib()
        saved = {k: os.environ.get(k) for k in (env or {})}
        os.environ.update(env or {})  # plan knobs are read at plan creation
        try:
            self.plan = _native.Plan(ns_loc, nobs_loc, n, dev.index)
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        if comm is not None:
            st = _native.EnkfStatus()
            _native.raise_for_status(self.lib.enkf_plan_set_comm(self.plan.handle, comm.handle, ctypes.byref(st)),
                                     st, "enkf_plan_set_comm")
        self.lib.enkf_debug_set_stage_events.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        self.lib.enkf_debug_stage_times.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]
        self.lib.enkf_debug_set_gram_events.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        self.lib.enkf_debug_gram_times.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]

    def step(self, x, y, idx, r, out, stream):
        code = self.lib.enkf_analysis_async_f64(self.plan.handle, x.data_ptr(), y.data_ptr(),
                                                0 if idx is None else idx.data_ptr(), r.data_ptr(),
                                                out.data_ptr(), stream)
        if code != 0:
            self.check(stream)
            raise RuntimeError(f"enkf_analysis_async_f64 returned {code}")

    def check(self, stream):
        st = self.native.EnkfStatus()
        code = self.lib.enkf_plan_sync_status(self.plan.handle, stream, self.ctypes.byref(st))
        self.native.raise_for_status(code, st, "analysis step")

    def stage_times(self, run_step, sync, reps=3):
        """ms of the gram | allreduce | levels | anomaly stages (library events)."""
        acc = [0.0] * 4
        self.lib.enkf_debug_set_stage_events(self.plan.handle, 1)
        for _ in range(reps):
            run_step()
            sync()
            four = (self.ctypes.c_float * 4)()
            if self.lib.enkf_debug_stage_times(self.plan.handle, four) == 0:
                for i in range(4):
                    acc[i] += four[i] / reps
        self.lib.enkf_debug_set_stage_events(self.plan.handle, 0)
        return dict(zip(("gram", "allreduce", "levels", "anomaly"), acc))

    def gram_pass_times(self, run_step, sync, reps=3):
        acc = [0.0, 0.0]
        self.lib.enkf_debug_set_gram_events(self.plan.handle, 1)
        for _ in range(reps):
            run_step()
            sync()
            two = (self.ctypes.c_float * 2)()
            if self.lib.enkf_debug_gram_times(self.plan.handle, two) == 0:
                acc[0] += two[0] / reps
                acc[1] += two[1] / reps
        self.lib.enkf_debug_set_gram_events(self.plan.handle, 0)
        return acc


def small_problem(cfg):
    from paper_1302_3876_b200 import workloads as W
    return {1: W.config1, 2: lambda: W.Config2Cycler().cycle(), 3: W.config3}[cfg]()


def run_config2_cycles(dev, cycles=100, reps=3):
    """Config 2's 100-cycle closed loop (experiment.py:457-479 with the Lorenz-96
    model): perturbed observations of a seeded truth trajectory pre-staged on the
    device, the whole loop in one call (forecast -> analysis per cycle, one
    synchronisation); best of `reps`.  The oracle's loop on the host over 5 cycles."""
    import numpy as np
    import torch

    import oracle
    import paper_1302_3876_b200 as P
    from paper_1302_3876_b200 import workloads as W

    cyc = W.Config2Cycler()
    ns, nens = cyc.ns, cyc.nens
    truth = cyc.truth.copy()
    rng = W.make_rng(0xC2)
    ys = []
    for _ in range(cycles):
        for _ in range(5):
            truth = W.l96_rk4(truth)
        y = truth + 0.1 * rng.standard_normal(ns)
        ys.append(y[:, None] + 0.1 * rng.standard_normal((ns, nens)))
    ys_d = torch.from_numpy(np.stack(ys)).to(dev)
    x0 = torch.from_numpy(cyc.x).to(dev)
    r = np.full(ns, 0.01)
    model = P.Lorenz96(P.Lorenz96Config(nstate=ns))
    P.cycle_l96(model, x0, ys_d, P.SelectionOperator.identity(), r, 5)  # warm
    best = float("inf")
    for _ in range(reps):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        res = P.cycle_l96(model, x0, ys_d, P.SelectionOperator.identity(), r, 5)
        torch.cuda.synchronize(dev)
        best = min(best, time.perf_counter() - t0)
    assert bool(torch.isfinite(res.mean_a).all())
    t0 = time.perf_counter()
    oracle.cycle_l96(cyc.x, np.stack(ys[:5]), None, r, 5)
    cpu = (time.perf_counter() - t0) / 5
    return {"cycles": cycles, "cycles_per_s": cycles / best, "ms_per_cycle": best / cycles * 1e3,
            "api": "paper_1302_3876_b200.cycle_l96 (device-resident loop, one call)",
            "cpu_oracle_ms_per_cycle": cpu * 1e3}


def timed_steps(run_step, steps, dev, stream, world, dist):
    import torch
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(steps):
        run_step()
    stop.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(stop)
    if world > 1:
        mt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
        ms = float(mt.item())
    return ms


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1302_3876_b200 import workloads as W
    from paper_1302_3876_b200.build import build

    world, rank, local = dist_env()
    nccl_dir = None
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        nccl_dir = nccl_log_setup()
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()

    cfg, scale = args.config, args.scale_log2
    z = W.SIZES[cfg]
    small = cfg <= 3
    if small:
        p = small_problem(cfg)
        ns, nobs, n = p.shape
        indices = p.indices
    else:
        ns, nobs, n = z["ns"] >> scale, z["nobs"] >> scale, z["nens"]
        indices = W.random_indices(ns, nobs / ns, W.SEEDS[cfg]["h"])
    shard_world = 1 if small else world  # configs 1-3 do not shard: N independent replicas

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sl = args.cpu_sample_log2 if args.cpu_sample_log2 is not None else cpu_sample_log2(cfg, scale)
        cpu = run_cpu_oracle(cfg, scale, sl, steps=2, warmup=0 if not small else 1)

    if small:
        x = torch.from_numpy(p.x).to(dev)
        yv = torch.from_numpy(p.perturbed).to(dev)
        r = torch.from_numpy(p.r).to(dev)
        idx = None if p.indices is None else torch.from_numpy(p.indices).to(dev)
    else:
        shard = W.device_problem_shard(cfg, world, rank, dev, scale, indices=indices)
        x, yv, r, idx = shard["x"], shard["perturbed"], shard["r"], shard["idx"]
    ns_loc, nobs_loc = x.shape[0], yv.shape[0]
    xa = torch.empty_like(x)
    comm = None
    if shard_world > 1:
        from paper_1302_3876_b200.distributed import NativeComm
        comm = NativeComm(dev)
    runner = Runner(ns_loc, nobs_loc, n, dev, comm)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    def step():
        runner.step(x, yv, idx, r, xa, sptr)

    for _ in range(args.warmup):
        step()
    runner.check(sptr)
    # Large configs: the library records its stage-boundary events during the timed
    # steps themselves (5 cudaEventRecord per 9-45 ms step, into a ring of 64 event sets),
    # so `kernels_ms` and the rooflines are the MEAN over the timed steps (the last 64 at
    # most), measured inside the timed region in its steady power state.  Small configs
    # (tens of microseconds per step) keep the events out of the timed region.
    stage_in_region = not small
    if stage_in_region:
        runner.lib.enkf_debug_set_stage_events(runner.plan.handle, 1)
    with ClockSampler(local) as clocks, EnergyMeter(local) as energy:
        ms = timed_steps(step, args.steps, dev, stream, world, dist)
    runner.check(sptr)
    sync = lambda: torch.cuda.synchronize(dev)  # noqa: E731

    stages = None
    stage_steps = 0
    if stage_in_region:
        import ctypes
        four = (ctypes.c_float * 4)()
        nst = ctypes.c_int32(0)
        runner.lib.enkf_debug_stage_times_mean.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_float),
                                                           ctypes.POINTER(ctypes.c_int32)]
        if runner.lib.enkf_debug_stage_times_mean(runner.plan.handle, four, ctypes.byref(nst)) == 0:
            stages = dict(zip(("gram", "allreduce", "levels", "anomaly"), (float(v) for v in four)))
            stage_steps = int(nst.value)
        runner.lib.enkf_debug_set_stage_events(runner.plan.handle, 0)
    if stages is None:
        stage_in_region = False
        stages = runner.stage_times(step, sync)
    if not any(stages.values()):  # config 1: the whole step is one single-CTA kernel (tiny.cuh)
        stages = {"analysis_tiny": ms / args.steps}
    gram_i8 = n == 128 and os.environ.get("ENKF_GRAM", "i8ls") != "fp64" and not small
    passes = runner.gram_pass_times(step, sync) if (gram_i8 and not args.no_extras) else None
    stages_all = None
    if world > 1:
        tv = torch.tensor([stages[k] for k in ("gram", "allreduce", "levels", "anomaly")], dtype=torch.float64,
                          device=dev)
        gath = [torch.empty_like(tv) for _ in range(world)]
        dist.all_gather(gath, tv)
        stages_all = [[round(float(v), 4) for v in g.cpu()] for g in gath]

    # ---- the strict IEEE-FP64 step (DMMA Gram + DMMA anomaly update), same run
    strict = None
    if not args.no_extras and n == 128:
        r64 = Runner(ns_loc, nobs_loc, n, dev, comm, env={"ENKF_GRAM": "fp64", "ENKF_ANOMALY": "fp64"})

        def step64():
            r64.step(x, yv, idx, r, xa, sptr)
        for _ in range(max(1, args.warmup)):
            step64()
        r64.check(sptr)
        with ClockSampler(local) as clocks64, EnergyMeter(local) as energy64:
            ms64 = timed_steps(step64, args.steps, dev, stream, world, dist)
        r64.check(sptr)
        st64 = r64.stage_times(step64, sync)
        cs = clocks64.summary()
        strict = {"value": args.steps / (ms64 / 1e3), "unit": "steps/s", "ms_per_step": ms64 / args.steps,
                  "dtype": "f64 (IEEE: FP64 DMMA m8n8k4 Gram + FP64 DMMA anomaly update)",
                  "kernels_ms": st64, "clocks": cs,
                  "energy_j_per_step": energy64.joules / args.steps if energy64.joules else None,
                  "env": "ENKF_GRAM=fp64 ENKF_ANOMALY=fp64"}
        del r64

    # ---- overflow cliff: one Y element beyond its column's sampled scale sends the
    # int8 Gram to the flag-gated FP64 fallback (measured, then restored)
    cliff = None
    if gram_i8 and not args.no_extras and world == 1:
        k = nobs_loc // 3
        old = float(yv[k, 5])
        yv[k, 5] = 1e6
        st_f = runner.stage_times(step, sync)
        runner.check(sptr)
        yv[k, 5] = old
        step()
        runner.check(sptr)
        cliff = {"gram_ms_fallback": st_f["gram"], "gram_ms": stages["gram"],
                 "extra_ms": st_f["gram"] - stages["gram"],
                 "trigger": "one element of Y (or X[idx]) more than ~4x its column's sampled max "
                            "(G8_HEADROOM = 2 bits): the int8 Gram pass flags it and gram128_kernel (FP64 DMMA) "
                            "recomputes the Gram on the same stream"}

    # ---- config 2 as the configuration defines it: 100 closed-loop assimilation cycles
    # (5 RK4 steps + one analysis each) device-resident (enkf_cycle_l96_f64), against
    # the oracle's loop on the host
    cycled = None
    if cfg == 2 and not args.no_extras and rank == 0:
        cycled = run_config2_cycles(dev)
    # latency-bound configs: the same step captured once into a CUDA graph and replayed
    # (the plan allocates its workspace at creation, so the capture needs no warm-up)
    graphed = None
    if small and not args.no_extras:
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            runner.step(x, yv, idx, r, xa, gs.cuda_stream)
        graph.replay()
        torch.cuda.synchronize(dev)
        runner.check(sptr)
        ms_g = timed_steps(graph.replay, args.steps, dev, torch.cuda.current_stream(dev), 1, dist)
        runner.check(sptr)
        graphed = {"value": args.steps / (ms_g / 1e3), "unit": "steps/s", "ms_per_step": ms_g / args.steps,
                   "api": "enkf_analysis_async_f64 captured into a CUDA graph, replayed"}
        del graph

    # ---- e2e with host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        import paper_1302_3876_b200 as P
        x_h = torch.empty(tuple(x.shape), dtype=torch.float64, pin_memory=True)
        y_h = torch.empty(tuple(yv.shape), dtype=torch.float64, pin_memory=True)
        x_h.copy_(x)
        y_h.copy_(yv)
        r_h = r.cpu().numpy()
        idx_loc = None if idx is None else idx.cpu().numpy()
        del x, xa, yv
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()
        if shard_world == 1:
            h = P.SelectionOperator.identity() if idx_loc is None else P.SelectionOperator.from_indices(idx_loc)
            obs = P.ObservationBatch(y=None, perturbed=y_h.numpy(), perturbations=None)
            xnp = x_h.numpy()

            def e2e_step():
                return P.analysis_step(xnp, obs, h, r_h)  # numpy in, numpy out
            api = "paper_1302_3876_b200.analysis_step(numpy host arrays) -> enkf_analysis_host_f64"
        else:
            from paper_1302_3876_b200.distributed import NativeShardedAnalysis
            shard_runner = NativeShardedAnalysis(ns_loc, nobs_loc, n, dev, comm)
            out_h = torch.empty_like(x_h, pin_memory=True).numpy()
            xnp, ynp = x_h.numpy(), y_h.numpy()

            def e2e_step():
                return shard_runner.step_host(xnp, ynp, idx_loc, r_h, out_h)
            api = ("paper_1302_3876_b200.distributed.NativeShardedAnalysis.step_host (pinned host shards) -> "
                   "enkf_analysis_host_f64 with the NCCL communicator attached")
        e2e_step()  # warm (plans, staging)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        el = time.perf_counter() - t0
        if world > 1:
            et = torch.tensor([el], dtype=torch.float64, device=dev)
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
            el = float(et.item())
        streamed = (shard_world == 1 and idx_loc is not None and os.environ.get("ENKF_HOST_STREAM", "1") != "0"
                    and x_h.numel() * 8 > (1 << 20))
        e2e = {"value": args.e2e_steps / el, "unit": "steps/s",
               # streamed host path: the observed rows X[idx] cross PCIe twice (the
               # gather that feeds the Gram pass, then with their X chunk)
               "h2d_bytes_per_step": int(x_h.numel() * 8 + y_h.numel() * 8 + r_h.nbytes
                                         + (idx_loc.nbytes if idx_loc is not None else 0)
                                         + (y_h.numel() * 8 if streamed else 0)) * shard_world,
               "d2h_bytes_per_step": int(x_h.numel() * 8) * shard_world, "steps": args.e2e_steps,
               "inputs": "page-locked host buffers (pageable inputs take the staging-ring path)",
               "api": api}

    nccl_lines = nccl_init_lines(nccl_dir) if rank == 0 else None
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    steps_per_s = args.steps / (ms / 1e3)
    ms_step = ms / args.steps
    peak, peak_src = hbm_peak()
    t_anom = stages.get("anomaly", ms_step) or ms_step
    t_gram = stages.get("gram", 0.0)
    bytes_anom = 2.0 * ns_loc * n * 8
    anom_gbs = bytes_anom / (t_anom * 1e-3) / 1e9
    flop_anom = 2.0 * ns_loc * n * n
    anom_tflops = flop_anom / (t_anom * 1e-3) / 1e12
    tensor_core = n == 128 and os.environ.get("ENKF_ANOMALY", "i8") != "fp64"
    if tensor_core:
        traffic, traffic_src = None, None
        try:  # DRAM bytes per row from the committed ncu --set full capture, times this launch's rows
            cap = json.load(open(os.path.join(ROOT, "profiles", "r01_anomaly_dram.json")))
            traffic = cap["dram_bytes_per_row"] * ns_loc
            traffic_src = ("dram__bytes_read.sum + dram__bytes_write.sum per row from " + cap["capture"] +
                           f", x {ns_loc} rows per launch ({cap['ratio_to_algorithmic']:.4f} x algorithmic)")
        except (OSError, KeyError, ValueError):
            pass
        roofline = {"bound": "hbm", "kernel": "anomaly_i8_kernel (X^A = X T, tcgen05.mma kind::i8 on exact byte digits, TMA-staged)",
                    "achieved": anom_gbs, "peak": peak, "unit": "GB/s", "frac": anom_gbs / peak,
                    "traffic": traffic, "traffic_source": traffic_src,
                    "algorithmic": f"read X + write X^A = 2*n_state*n_ens*8 = {bytes_anom:.3e} B per launch",
                    "peak_source": peak_src,
                    "fp64_view": {"equivalent_tflops": anom_tflops, "fp64_dmma_peak": FP64_DMMA_PEAK_TFLOPS,
                                  "frac": anom_tflops / FP64_DMMA_PEAK_TFLOPS}}
    else:
        roofline = {"bound": "tensor", "kernel": "rowgemm_ws_kernel (X^A = X T, FP64 DMMA)",
                    "achieved": anom_tflops, "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": anom_tflops / FP64_DMMA_PEAK_TFLOPS, "traffic": None,
                    "algorithmic": f"2*n_state*n_ens^2 = {flop_anom:.3e} flop per launch",
                    "peak_source": "measured FP64 DMMA m8n8k4 issue rate on this pool's B200 (profiles/r01_fp64_probe.json); MEASURED_PEAKS.json has no FP64 entry",
                    "hbm_view": {"achieved_gbs": anom_gbs, "peak_gbs": peak, "frac": anom_gbs / peak}}
    if small:
        roofline["note"] = "configs 1-3 are launch/latency-bound (SURVEY §8(d)); the fraction is reported, not a target"

    # the whole step on its compulsory bytes (SURVEY §8(d) B_step)
    b_step = 8.0 * (2 * ns * n + 2 * nobs * n + 2 * nobs)
    f_step = 6.0 * (n * n * nobs + n * nobs) + 2.0 * n * n * nobs + 2.0 * n * n * ns
    t_floor = max(b_step / (peak * shard_world * 1e9), f_step / (FP64_DMMA_PEAK_TFLOPS * shard_world * 1e12))
    roofline_step = {"bound": "hbm", "unit": "GB/s", "bytes": b_step,
                     "achieved": b_step / (ms_step * 1e-3) / 1e9, "peak": peak * shard_world,
                     "frac": b_step / (ms_step * 1e-3) / 1e9 / (peak * shard_world),
                     "algorithmic": "B_step = 8*(2*Ns*N + 2*Nobs*N + 2*Nobs): read X, write X^A, read X[idx] rows, Y, r, idx",
                     # achieved = max(B_step / P_hbm, F_step / P_fp64) / t_step, with
                     # F_step = 6(N^2 Nobs + N Nobs) + 2 N^2 Nobs + 2 N^2 Ns; > 1 means faster than an
                     # FP64 implementation could be (the int8-digit emulation)
                     "survey_formula": {"f_step_flop": f_step, "floor_ms": t_floor * 1e3,
                                        "achieved": t_floor / (ms_step * 1e-3),
                                        "p_fp64_tflops": FP64_DMMA_PEAK_TFLOPS}}

    ism = None
    comp_row = 2 * n * 8 + 16
    if passes is not None:
        ratio = None
        try:
            cap = json.load(open(os.path.join(ROOT, "profiles", "r01_gram_dram.json")))
            ratio = cap["ratio_to_compulsory"]
        except (OSError, KeyError, ValueError):
            pass
        ism = {"kernel": "gram_i8_slice_kernel: the observation-row streaming pass of the Gram (reduced-coordinate "
                         "ISM, DESIGN §3/§6), which replaces the reference's per-group sweeps of the Nobs x 2N panel",
               "bound": "hbm", "unit": "GB/s", "ms": passes[0],
               "achieved": nobs_loc * comp_row / (passes[0] * 1e-3) / 1e9, "peak": peak,
               "frac": nobs_loc * comp_row / (passes[0] * 1e-3) / 1e9 / peak,
               "algorithmic": f"compulsory bytes per observed row: read X[idx] row and Y row (2*N*8 B), r and idx "
                              f"(16 B) = {comp_row} B",
               "traffic_ratio": ratio,
               "traffic_source": "whole Gram (slice + MMA passes) DRAM bytes / compulsory, ncu --set full "
                                 "(profiles/r01_gram_dram.json)",
               "mma_pass_ms": passes[1]}
    gram_compulsory = nobs_loc * comp_row / (t_gram * 1e-3) / 1e9 if t_gram > 0 else None
    flop_gram = 2.0 * nobs_loc * n * (2 * n)
    cs = clocks.summary()
    # our kernels per step: Gram (int8: scales, slice, MMA, reduce + the two flag-gated
    # FP64-fallback kernels, which exit at once | FP64: gram128 + reduce | tiny: 1 kernel
    # for the whole step), levels, anomaly; + flag pack/unpack around the NCCL allreduce
    if small and cfg == 1:
        per_step = 1
    else:
        per_step = (6 if gram_i8 else 2) + 2 + (2 if comm is not None else 0)
    line = {
        "metric": "EnKF analysis steps/sec",
        "value": steps_per_s,
        "unit": "steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong" if not small else "replicas",
        "vs_baseline": None,
        "dtype": EMULATED_DTYPE if (tensor_core or gram_i8) else "f64",
        "data": ("synthetic (config value distributions, drawn on device with torch Philox; H indices from the "
                 "reference's seeded Philox draw)" if not small else
                 "synthetic (host numpy Philox: the configuration's own generator, tests/golden pinned)"),
        "config": {"workload": workload_name(cfg, scale), "n_state": ns, "n_obs": nobs, "n_ens": n,
                   "parallelism": (f"row-shard x{world} (one ncclAllReduce of the {n}x{2 * n} Gram + flags per step, "
                                   "issued by libenkf_b200 on the compute stream)") if shard_world > 1 else
                   ("single GPU" if world == 1 else f"{world} independent replicas"),
                   "l2": ("inputs larger than L2 (X is %.0f GiB per GPU)" % (ns_loc * n * 8 / 2**30)) if not small
                   else "inputs L2-resident (latency-bound configuration)"},
        "kernels_ms": stages,
        "kernels_ms_source": (f"library stage events, mean over {stage_steps} timed steps (inside the timed region)"
                              if stage_in_region else
                              "library stage events of 3 extra steps after the timed region (averaged)"),
        "kernels_ms_per_rank": stages_all,
        "roofline": roofline,
        "roofline_step": roofline_step,
        "ism_sweep": ism,
        "gram_kernel": {"impl": ("gram_i8_slice_kernel + gram_i8_mma_ls_kernel (level split, N = 256 MMAs) "
                                 "(exact byte-digit products on tcgen05 kind::i8; ENKF_GRAM=fp64 selects the "
                                 "FP64 DMMA gram128_kernel)") if gram_i8 else "FP64 DMMA Gram",
                        "hbm_gbs_compulsory": gram_compulsory,
                        "hbm_frac_compulsory": gram_compulsory / peak if gram_compulsory else None,
                        "fp64_equiv_tflops": flop_gram / (t_gram * 1e-3) / 1e12 if t_gram > 0 else None},
        "strict_fp64": strict,
        "overflow_cliff": cliff,
        "clocks": {k: cs[k] for k in ("sm_mhz", "sm_max_mhz", "reasons", "samples")},
        # board energy of the timed region from NVML's cumulative counter (this GPU);
        # the step runs at the ~1 kW power cap, so J/step is what bounds steps/s
        "energy_j_per_step": energy.joules / args.steps if energy.joules else None,
        "power_w": energy.joules / (ms / 1e3) if energy.joules else None,
        "energy_scope": "rank 0's GPU board (NVML total-energy counter over the timed region)",
        "gpu_launches": per_step * args.steps,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    if cycled is not None:
        line["cycled"] = cycled
    if graphed is not None:
        line["graph_replay"] = graphed
    if nccl_lines is not None:
        line["nccl_init"] = nccl_lines
        for ln in nccl_lines:
            print("[nccl] " + ln, file=sys.stderr)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg, scale = args.config, args.scale_log2
    sl = args.cpu_sample_log2 if args.cpu_sample_log2 is not None else cpu_sample_log2(cfg, scale)
    cpu = run_cpu_oracle(cfg, scale, sl, steps=min(args.steps, 5), warmup=min(args.warmup, 1))
    from paper_1302_3876_b200 import workloads as W
    z = W.SIZES[cfg]
    line = {
        "metric": "EnKF analysis steps/sec", "value": cpu["value"], "unit": "steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / cpu["value"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (host numpy Philox, same distributions)",
        "config": {"workload": workload_name(cfg, scale), "n_state": z["ns"] >> scale,
                   "n_obs": z["nobs"] >> scale, "n_ens": z["nens"], "parallelism": "host CPU"},
        "impl": "reference",
        "cpu_baseline": cpu,
        "e2e": {"value": cpu["value"], "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        # configs 4/5 do not fit a host-run of the full workload (config 5 needs ~300 GB and
        # minutes per step): each timed step is a row sample, the value the full-size
        # throughput extrapolated linearly (the `linearity` object shows two sample sizes)
        "extrapolated": bool(cpu.get("extrapolated")),
        "measured_seconds_per_sample_step": cpu.get("sample_seconds"),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    else:
        world, _, _ = dist_env()
        if world != args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), file=sys.stderr)
            sys.exit(2)
        run_ours(args)


if __name__ == "__main__":
    main()
