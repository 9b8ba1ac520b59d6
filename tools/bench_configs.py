"""Steps/s of the analysis step at every BASELINE.json configuration (1 GPU),
device-resident (`enkf_analysis_f64` on CUDA tensors) and through the public
API with host numpy arrays, next to the CPU oracle on the same inputs.

    python tools/bench_configs.py [--configs 1,2,3,4] [--reps 20]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402  (CPU baseline: test/bench infrastructure)
import paper_1302_3876_b200 as P  # noqa: E402
from paper_1302_3876_b200 import workloads as W  # noqa: E402


def problem(cfg):
    if cfg == 1:
        return W.config1()
    if cfg == 2:
        return W.Config2Cycler().cycle()
    if cfg == 3:
        return W.config3()
    if cfg == 4:
        return W.config4(0)
    raise ValueError(cfg)


def time_device(p, reps):
    dev = torch.device("cuda", 0)
    h = P.SelectionOperator.identity() if p.indices is None else P.SelectionOperator.from_indices(p.indices)
    x = torch.from_numpy(p.x).to(dev)
    obs = P.ObservationBatch(y=None, perturbed=torch.from_numpy(p.perturbed).to(dev), perturbations=None)
    r = torch.from_numpy(p.r).to(dev)
    for _ in range(3):
        P.analysis_step(x, obs, h, r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        P.analysis_step(x, obs, h, r)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps
    return e0.elapsed_time(e1) / reps / 1e3, wall


def time_host(p, reps):
    h = P.SelectionOperator.identity() if p.indices is None else P.SelectionOperator.from_indices(p.indices)
    obs = P.ObservationBatch(y=p.y, perturbed=p.perturbed, perturbations=None)
    P.analysis_step(p.x, obs, h, p.r)
    xa = None
    t0 = time.perf_counter()
    for _ in range(reps):
        xa = None  # drop the previous result first: its page-locked block is reused
        xa = P.analysis_step(p.x, obs, h, p.r)
    dt = (time.perf_counter() - t0) / reps
    return dt, xa


def time_oracle(p, reps):
    oracle.analysis_step(p.x, p.perturbed, p.indices, p.r)
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        xa = oracle.analysis_step(p.x, p.perturbed, p.indices, p.r)
        best = min(best, time.perf_counter() - t0)
    return best, xa


def time_cycled(cycles=100, cpu_cycles=5):
    """Config 2 as the reference runs it: closed-loop cycles of 5 RK4 steps +
    one analysis, device-resident (cycle_l96) vs the CPU oracle loop."""
    cyc = W.Config2Cycler()
    ns, nens = cyc.ns, cyc.nens
    rng = np.random.Generator(np.random.Philox(0xC2))
    ys = cyc.x.mean(axis=1)[None, :, None] + 0.1 * rng.standard_normal((cycles, ns, nens))
    r = np.full(ns, 0.01)
    model = P.Lorenz96(P.Lorenz96Config(nstate=ns))
    h = P.SelectionOperator.identity()
    dev = torch.device("cuda", 0)
    x0 = torch.from_numpy(cyc.x).to(dev)
    yd = torch.from_numpy(ys).to(dev)
    P.cycle_l96(model, x0, yd[:3], h, r, 5)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.cycle_l96(model, x0, yd, h, r, 5)
    torch.cuda.synchronize()
    gpu_s = (time.perf_counter() - t0) / cycles
    t0 = time.perf_counter()
    oracle.cycle_l96(cyc.x, ys[:cpu_cycles], None, r, 5)
    cpu_s = (time.perf_counter() - t0) / cpu_cycles
    return {"config2_cycled": {"cycles": cycles, "gpu_cycles_per_s": 1.0 / gpu_s, "gpu_ms_per_cycle": gpu_s * 1e3,
                               "cpu_oracle_cycles_per_s": 1.0 / cpu_s, "cpu_sample_cycles": cpu_cycles,
                               "cpu_threads": os.cpu_count(), "note": "wall clock incl. one sync per 100 cycles"}}


def time_lorenz_small(cycles=200):
    """The lorenz-small preset's assimilation loop (presets/lorenz-small.ini: 40 states,
    20 members, all observed, R = I, analysis every 2 RK4 steps for 400 steps, inflation
    1.05, cyclic localization scale 8) on the device (cycle_l96, localized) vs the CPU
    oracle loop, on the golden fixture's first ensemble and staged observations."""
    from golden_io import load
    g = load("lorenz96")
    x0, r = g["lcA_x0"], g["lcA_r"]
    rng = np.random.Generator(np.random.Philox(0x51))
    ys = x0.mean(axis=1)[None, :, None] + rng.standard_normal((cycles, x0.shape[0], x0.shape[1]))
    model = P.Lorenz96(P.Lorenz96Config(nstate=x0.shape[0]))
    h = P.SelectionOperator.identity()
    P.cycle_l96(model, x0, ys[:2], h, r, 2, inflation=1.05, localization_scale=8.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.cycle_l96(model, x0, ys, h, r, 2, inflation=1.05, localization_scale=8.0)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    xo, _, _ = oracle.cycle_l96(x0, ys, None, r, 2, inflation=1.05, localization_scale=8.0)
    cpu_s = time.perf_counter() - t0
    err = float(np.abs(res.x.cpu().numpy() - xo).max() / np.abs(xo).max())
    return {"lorenz_small_loop": {"cycles": cycles, "gpu_s": gpu_s, "gpu_ms_per_cycle": gpu_s / cycles * 1e3,
                                  "cpu_oracle_s": cpu_s, "cpu_threads": os.cpu_count(), "xa_rel_err_vs_oracle": err}}


def time_localized(reps=5):
    """Localized analysis (enkf.py:193-199): GPU matrix-free cyclic
    influence (taper evaluated in-kernel), GPU with the dense influence matrix, and the
    CPU oracle with the dense matrix, on a small, a config-2-sized and a larger case."""
    out = {}
    cases = [("l96_40", 40, 20, 20, 10.0), ("l96_4096", 4096, 64, 2048, 50.0), ("ns65536", 1 << 16, 128, 1 << 13, 500.0)]
    for name, ns, nens, nobs, scale in cases:
        rng = np.random.Generator(np.random.Philox(ns + nens))
        x = rng.standard_normal((ns, nens)) * rng.uniform(0.5, 2.0, (ns, 1)) + rng.standard_normal((ns, 1))
        idx = np.sort(rng.choice(ns, size=nobs, replace=False))
        r = rng.uniform(0.25, 1.0, nobs)
        pert = x[idx].mean(axis=1)[:, None] + rng.standard_normal((nobs, nens))
        h = P.SelectionOperator.from_indices(idx)
        obs = P.ObservationBatch(y=None, perturbed=pert, perturbations=None)
        lazy = P.influence_matrix_cyclic(ns, h, scale=scale)
        dense = np.asarray(lazy)
        dev = torch.device("cuda", 0)
        xd, rd = torch.from_numpy(x).to(dev), torch.from_numpy(r).to(dev)
        obs_d = P.ObservationBatch(y=None, perturbed=torch.from_numpy(pert).to(dev), perturbations=None)
        dd = torch.from_numpy(dense).to(dev)
        res = {"shape": {"n_state": ns, "n_ens": nens, "n_obs": nobs, "scale": scale}}
        for key, loc in (("gpu_matrix_free_ms", lazy), ("gpu_dense_ms", dd)):
            P.analysis_step(xd, obs_d, h, rd, "sherman", localization=loc)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(reps):
                xa = P.analysis_step(xd, obs_d, h, rd, "sherman", localization=loc)
            torch.cuda.synchronize()
            res[key] = (time.perf_counter() - t0) / reps * 1e3
        t0 = time.perf_counter()
        ref = oracle.analysis_step_localized(x, pert, idx, r, dense)
        res["cpu_oracle_dense_ms"] = (time.perf_counter() - t0) * 1e3
        res["xa_rel_err_vs_oracle"] = float(np.abs(xa.cpu().numpy() - ref).max() / np.abs(ref).max())
        out[name] = res
    return {"localized": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--cycled", action="store_true", help="also time the config-2 closed loop")
    ap.add_argument("--localized", action="store_true", help="also time the localized analysis (row f4)")
    a = ap.parse_args()
    out = {}
    if a.cycled:
        print(json.dumps(time_cycled()), flush=True)
        print(json.dumps(time_lorenz_small()), flush=True)
    if a.localized:
        print(json.dumps(time_localized()), flush=True)
    for cfg in [int(c) for c in a.configs.split(",") if c]:
        p = problem(cfg)
        reps = a.reps if cfg < 4 else 3
        dev_s, dev_wall = time_device(p, reps)
        host_s, xa = time_host(p, reps if cfg < 4 else 2)
        cpu_s, ref = time_oracle(p, 3 if cfg < 4 else 1)
        err = float(np.abs(xa - ref).max() / np.abs(ref).max())
        out[f"config{cfg}"] = {
            "shape": {"n_state": p.shape[0], "n_obs": p.shape[1], "n_ens": p.shape[2]},
            "device_steps_per_s": 1.0 / dev_s, "device_ms": dev_s * 1e3, "device_wall_ms": dev_wall * 1e3,
            "host_api_steps_per_s": 1.0 / host_s, "host_api_ms": host_s * 1e3,
            "cpu_oracle_steps_per_s": 1.0 / cpu_s, "cpu_oracle_ms": cpu_s * 1e3, "cpu_threads": os.cpu_count(),
            "xa_rel_err_vs_oracle": err,
        }
        print(json.dumps({f"config{cfg}": out[f"config{cfg}"]}), flush=True)


if __name__ == "__main__":
    main()
