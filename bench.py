"""Benchmark of the B200 EnKF analysis step (iterative Sherman-Morrison).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

N > 1 runs under torchrun (one rank per GPU, NCCL).  One JSON line on rank 0.

A "step" = one full analysis step (BASELINE.json metric "EnKF analysis
steps/sec"): level-0 Gram pass over the observed rows, NCCL allreduce of the
N x 2N Gram (N > 1), the N Sherman-Morrison levels, and the anomaly update
X^A = X T over every state row.  Workload = config 5 (n_state = 2^26,
n_ens = 128, n_obs = 2^23) by default: the config BASELINE.json's 1/2/4/8-GPU
scaling is quoted on; it fits one B200 (X + X^A + Y = 136 GiB).

  value : steps/s, whole job, inputs resident in HBM, CUDA-event timed,
          max over ranks (strong scaling: the problem is fixed, rows sharded).
  e2e   : the same metric through the public API `analysis_step` with host
          numpy buffers, host->device and device->host copies inside.
  roofline : the anomaly-update kernel (the dominant one).  For n_ens = 128
          it runs on the tcgen05 int8 tensor cores (exact byte-digit split of
          the fp64 product) and is HBM-bound: GB/s of X read + X^A written
          against MEASURED_PEAKS.json.  ENKF_ANOMALY=fp64 selects the FP64
          DMMA kernel (FP64 TFLOP/s against the measured DMMA peak).
  cpu_baseline : the CPU oracle (oracle/, a numpy/OpenBLAS restatement of the
          reference, which is pure Python) on a bounded row sample of the same
          workload, scaled linearly to the full size (cost is linear in
          n_state and n_obs at fixed n_ens).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_DMMA_PEAK_TFLOPS = 37.07  # measured: profiles/r01_fp64_probe.json (DMMA m8n8k4, 148 SMs)
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[4, 5])
    ap.add_argument("--scale-log2", type=int, default=0, help="shrink n_state/n_obs by 2^s (testing)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
    return (f"config{cfg}: n_state=2^{(z['ns'] >> s).bit_length() - 1} n_ens={z['nens']} "
            f"n_obs=2^{(z['nobs'] >> s).bit_length() - 1}")


# ----------------------------------------------------------------------------- CPU legs
def cpu_sample_log2(cfg: int, scale: int) -> int:
    return {4: 6, 5: 8}[cfg] - scale if cfg in (4, 5) else 0


def run_cpu_oracle(cfg, scale, sample_log2, steps, warmup):
    """Time the oracle port (numpy + OpenBLAS, all host threads) on a row sample."""
    import numpy as np

    import oracle
    from paper_1302_3876_b200 import workloads as W

    s = max(0, sample_log2)
    p = (W.config4 if cfg == 4 else W.config5)(scale + s)
    for _ in range(warmup):
        oracle.analysis_step_chunked(p.x, p.perturbed, p.indices, p.r)
    times = []
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        oracle.analysis_step_chunked(p.x, p.perturbed, p.indices, p.r)
        times.append(time.perf_counter() - t0)
    t = min(times)
    factor = 2 ** s
    value = 1.0 / (t * factor)
    ns, nobs, n = p.shape
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    return dict(value=value, unit="steps/s", cores=int(threads), kind="port",
                sample=(f"oracle/ (numpy+OpenBLAS restatement of enkf.analysis_step) on a 1/{factor} "
                        f"row sample (n_state={ns}, n_obs={nobs}, n_ens={n}), best of {len(times)}: "
                        f"{t:.3f} s; value = 1/({t:.3f} s x {factor})"),
                sample_seconds=t)


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
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- GPU leg
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1302_3876_b200 import workloads as W
    from paper_1302_3876_b200.build import build

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()

    cfg, scale = args.config, args.scale_log2
    z = W.SIZES[cfg]
    ns, nobs, n = z["ns"] >> scale, z["nobs"] >> scale, z["nens"]
    indices = W.random_indices(ns, nobs / ns, W.SEEDS[cfg]["h"])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sl = args.cpu_sample_log2 if args.cpu_sample_log2 is not None else cpu_sample_log2(cfg, scale)
        cpu = run_cpu_oracle(cfg, scale, sl, steps=2, warmup=0)

    shard = W.device_problem_shard(cfg, world, rank, dev, scale, indices=indices)
    x, yv, r, idx = shard["x"], shard["perturbed"], shard["r"], shard["idx"]
    ns_loc, nobs_loc = x.shape[0], yv.shape[0]
    xa = torch.empty_like(x)
    from paper_1302_3876_b200.distributed import CudaStages, ShardedAnalysis
    runner = ShardedAnalysis(CudaStages(ns_loc, nobs_loc, n, dev))
    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        runner.step(x, yv, idx, r, xa, check=False, events=ev)

    for _ in range(args.warmup):
        step()
    runner.raise_for_status()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record(stream)
        for k in range(args.steps):
            step(evs[k])
        stop.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(stop)
    runner.raise_for_status()
    t_gram = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    t_ar = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    t_lev = sum(e[2].elapsed_time(e[3]) for e in evs) / args.steps
    t_anom = sum(e[3].elapsed_time(e[4]) for e in evs) / args.steps
    if world > 1:
        mt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
        ms = float(mt.item())

    # --- the Gram's two passes timed apart (int8 form): CUDA events recorded by the
    # library around the slice pass (the HBM-streaming pass that replaces the
    # reference's ISM sweep) and the MMA pass, over 3 extra steps after the timed region
    sweep_ms = None
    n_ens_ = n
    if n_ens_ == 128 and os.environ.get("ENKF_GRAM", "i8ls") in ("i8", "i8ls"):
        import ctypes
        from paper_1302_3876_b200 import _native
        lib = _native.lib()
        lib.enkf_debug_set_gram_events.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        lib.enkf_debug_gram_times.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]
        handle = runner.stages.plan.handle
        lib.enkf_debug_set_gram_events(handle, 1)
        acc = [0.0, 0.0]
        for _ in range(3):
            step()
            torch.cuda.synchronize(dev)
            two = (ctypes.c_float * 2)()
            if lib.enkf_debug_gram_times(handle, two) == 0:
                acc[0] += two[0] / 3
                acc[1] += two[1] / 3
        lib.enkf_debug_set_gram_events(handle, 0)
        sweep_ms = acc

    # --- e2e with host buffers, copies inside the timed region.  One GPU: the
    # public drop-in `analysis_step(numpy arrays)`; N GPUs: the public sharded
    # API (`distributed.ShardedAnalysis`) fed from each rank's host shard.
    e2e = None
    if not args.no_e2e:
        import paper_1302_3876_b200 as P
        x_h = torch.empty(tuple(x.shape), dtype=torch.float64, pin_memory=True)
        y_h = torch.empty(tuple(yv.shape), dtype=torch.float64, pin_memory=True)
        x_h.copy_(x)
        y_h.copy_(yv)
        r_h = r.cpu().numpy()
        idx_loc = idx.cpu().numpy()
        del x, xa, yv
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()
        if world == 1:
            h = P.SelectionOperator.from_indices(idx_loc)
            obs = P.ObservationBatch(y=None, perturbed=y_h.numpy(), perturbations=None)
            xnp = x_h.numpy()

            def e2e_step():
                out = P.analysis_step(xnp, obs, h, r_h)  # numpy in, numpy out
                return out
        else:
            out_h = torch.empty_like(x_h, pin_memory=True)
            r_d = torch.from_numpy(r_h).to(dev)
            idx_d = torch.from_numpy(idx_loc).to(dev)

            def e2e_step():
                xd = x_h.to(dev, non_blocking=True)
                yd = y_h.to(dev, non_blocking=True)
                runner.step(xd, yd, idx_d, r_d, xd)  # in place; raises on any rank's error
                out_h.copy_(xd)
                torch.cuda.synchronize(dev)
                return out_h
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
        e2e = {"value": args.e2e_steps / el, "unit": "steps/s",
               # world 1, pinned X: the observed rows X[idx] cross PCIe twice (the
               # gather that feeds the Gram pass, then with their X chunk)
               "h2d_bytes_per_step": int(x_h.numel() * 8 + y_h.numel() * 8 + r_h.nbytes + idx_loc.nbytes
                                         + (y_h.numel() * 8 if world == 1 and os.environ.get("ENKF_HOST_STREAM", "1") != "0"
                                            else 0)) * world,
               "d2h_bytes_per_step": int(x_h.numel() * 8) * world, "steps": args.e2e_steps,
               "api": ("paper_1302_3876_b200.analysis_step(numpy host arrays) -> enkf_analysis_host_f64" if world == 1
                       else "paper_1302_3876_b200.distributed.ShardedAnalysis.step from pinned host shards")}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    steps_per_s = args.steps / (ms / 1e3)
    flop_anom = 2.0 * ns_loc * n * n
    anom_tflops = flop_anom / (t_anom * 1e-3) / 1e12
    flop_gram = 2.0 * nobs_loc * n * (2 * n)
    gram_i8 = n == 128 and os.environ.get("ENKF_GRAM", "i8") != "fp64"
    bytes_anom = 2.0 * ns_loc * n * 8
    bytes_gram = nobs_loc * (2 * n * 8 + 16)
    try:
        peaks = json.load(open(PEAKS_PATH))
        hbm_peak, peak_src = float(peaks["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        hbm_peak, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    anom_gbs = bytes_anom / (t_anom * 1e-3) / 1e9
    tensor_core = n == 128 and os.environ.get("ENKF_ANOMALY", "i8") != "fp64"
    if tensor_core:
        # int8-digit tcgen05 kernel: the FP64 product is exact integer work on
        # the tensor cores; the kernel is bounded by streaming X in and X^A out
        traffic, traffic_src = None, None
        try:  # DRAM bytes per row from the committed ncu --set full capture, times this launch's rows
            cap = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                              "r01_anomaly_dram.json")))
            traffic = cap["dram_bytes_per_row"] * ns_loc
            traffic_src = ("dram__bytes_read.sum + dram__bytes_write.sum per row from " + cap["capture"] +
                           f", x {ns_loc} rows per launch ({cap['ratio_to_algorithmic']:.4f} x algorithmic)")
        except (OSError, KeyError, ValueError):
            pass
        roofline = {"bound": "hbm", "kernel": "anomaly_i8_kernel (X^A = X T, tcgen05.mma kind::i8 on exact byte digits, TMA-staged)",
                    "achieved": anom_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": anom_gbs / hbm_peak,
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
                    "hbm_view": {"achieved_gbs": anom_gbs, "peak_gbs": hbm_peak, "frac": anom_gbs / hbm_peak}}
    line = {
        "metric": "EnKF analysis steps/sec",
        "value": steps_per_s,
        "unit": "steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (config value distributions, drawn on device with torch Philox; H indices from the reference's seeded Philox draw)",
        "config": {"workload": workload_name(cfg, scale), "n_state": ns, "n_obs": nobs, "n_ens": n,
                   "parallelism": f"row-shard x{world} (NCCL allreduce of the {n}x{2*n} Gram)" if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (X is %.0f GiB per GPU)" % (ns_loc * n * 8 / 2**30)},
        "kernels_ms": {"gram": t_gram, "allreduce": t_ar, "levels": t_lev, "anomaly": t_anom},
        "roofline": roofline,
        "ism_sweep": None if sweep_ms is None else {
            "kernel": "gram_i8_slice_kernel: the observation-row streaming pass of the Gram (reduced-coordinate "
                      "ISM, DESIGN §3/§6), which replaces the reference's per-group sweeps of the Nobs x 2N panel",
            "bound": "hbm", "unit": "GB/s", "ms": sweep_ms[0],
            "achieved": nobs_loc * (2 * n * 8 + 16 + 2 * n * 6) / (sweep_ms[0] * 1e-3) / 1e9,
            "peak": hbm_peak, "frac": nobs_loc * (2 * n * 8 + 16 + 2 * n * 6) / (sweep_ms[0] * 1e-3) / 1e9 / hbm_peak,
            "algorithmic": "per observed row: read X[idx] row and Y row (2*N*8 B), r and idx (16 B), write its "
                           "6+6 byte-digit planes (2*N*6 B) = 3600 B",
            "mma_pass_ms": sweep_ms[1]},
        "gram_kernel": {"impl": ("gram_i8_slice_kernel + " +
                                 ("gram_i8_mma_kernel (column split)" if os.environ.get("ENKF_GRAM") == "i8"
                                  else "gram_i8_mma_ls_kernel (level split, N = 256 MMAs)") +
                                 " (exact byte-digit products on tcgen05 kind::i8; ENKF_GRAM=fp64 selects the "
                                 "FP64 DMMA gram128_kernel)") if gram_i8 else
                                "gram128_kernel (FP64 DMMA)",
                        "fp64_equiv_tflops": flop_gram / (t_gram * 1e-3) / 1e12 if t_gram > 0 else None,
                        "fp64_equiv_frac_of_dmma_peak": (flop_gram / (t_gram * 1e-3) / 1e12) / FP64_DMMA_PEAK_TFLOPS
                        if t_gram > 0 else None,
                        "hbm_gbs_compulsory": bytes_gram / (t_gram * 1e-3) / 1e9 if t_gram > 0 else None},
        "clocks": clocks.summary(),
        # kernels per step: Gram (int8: scales, slice, MMA, reduce + the two flag-gated
        # FP64-fallback kernels, which exit at once | FP64: gram128 + reduce); levels; anomaly
        "gpu_launches": ((6 if gram_i8 else 2) + 1 + 1) * args.steps,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg, scale = args.config, args.scale_log2
    sl = args.cpu_sample_log2 if args.cpu_sample_log2 is not None else cpu_sample_log2(cfg, scale)
    cpu = run_cpu_oracle(cfg, scale, sl, steps=args.steps, warmup=min(args.warmup, 1))
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
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
