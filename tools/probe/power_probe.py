"""Power / SM clock of each stage of the config-5 step run alone in a loop
(~3 s each), sampled with nvidia-smi: which kernel drives the sw_power_cap.

    python tools/probe/power_probe.py [scale_log2]
"""
import ctypes
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402
from paper_1302_3876_b200 import _native  # noqa: E402
from paper_1302_3876_b200 import workloads as W  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    dev = torch.device("cuda", 0)
    d = W.device_problem_shard(5, 1, 0, dev, scale_log2=scale)
    x, y, idx, r = d["x"], d["perturbed"], d["idx"], d["r"]
    ns, no, n = x.shape[0], y.shape[0], x.shape[1]
    lib = _native.lib()
    s = torch.cuda.current_stream().cuda_stream
    out = {}
    xa = torch.empty_like(x)
    modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["i8", "fp64"]
    for mode in modes:
        dbg = None
        if mode.startswith("dbg"):  # anomaly role skips (profiling only, wrong results;
            # needs a -DI8_DBG_BUILD variant: tools/build_variant.py dbg -DI8_DBG_BUILD, ENKF_LIB_VARIANT=dbg)
            dbg, mode = mode[3:], "i8"
            os.environ["ENKF_I8_DBG"] = dbg
        else:
            os.environ.pop("ENKF_I8_DBG", None)
        os.environ["ENKF_GRAM"] = mode
        plan = _native.Plan(ns, no, n, 0)
        gram = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)
        a = torch.empty((n, n), dtype=torch.float64, device=dev)
        t = torch.empty((n, n), dtype=torch.float64, device=dev)

        def gram_once():
            lib.enkf_ism_gram_f64(plan.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(),
                                  gram.data_ptr(), s)

        gram_once()
        lib.enkf_ism_levels_f64(plan.handle, gram.data_ptr(), a.data_ptr(), t.data_ptr(), None, s)

        def anomaly_once():
            lib.enkf_anomaly_update_f64(plan.handle, x.data_ptr(), t.data_ptr(), xa.data_ptr(), ns, s)

        stages = [("gram_" + mode, gram_once)] + ([("anomaly", anomaly_once)] if mode == "i8" else [])
        if mode == "i8" and dbg is None:
            stages.append(("plain_copy_X_to_XA", lambda: xa.copy_(x)))
        if dbg is not None:
            stages = [("anomaly_dbg" + dbg, anomaly_once)]
        for name, fn in stages:
            torch.cuda.synchronize()
            fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            one = time.perf_counter() - t0
            reps = max(3, int(3.0 / max(one, 1e-4)))
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with ClockSampler(0) as cs:
                ev0.record()
                for _ in range(reps):
                    fn()
                ev1.record()
                torch.cuda.synchronize()
            pw = [float(rw[3]) for rw in cs.rows if rw[3].replace(".", "").isdigit()]
            out[name] = {"ms": ev0.elapsed_time(ev1) / reps, "clocks": cs.summary(),
                         "power_w_median": sorted(pw)[len(pw) // 2] if pw else None}
            print(name, json.dumps(out[name]), flush=True)
        del plan


if __name__ == "__main__":
    main()
