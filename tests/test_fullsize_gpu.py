"""Full-size parity (BASELINE config 5: 2^26 states, 128 members, 2^23 observations,
the bench workload) through size-independent properties — the parity policy of
DESIGN.md §3: the oracle cannot run the 2^23-row observation-space solve inside a
test, and its own fp64 floor there is ~4e-9.

* the default product path (int8 tensor-core Gram + int8 anomaly update) against
  the all-FP64 DMMA path (`ENKF_GRAM=fp64 ENKF_ANOMALY=fp64`), two independent
  kernel families: Gram within 1e-13, A = V'Z and X^A within the north star's 1e-9
  (sampled rows exactly, every row through its member sum: a checksum per row);
* X^A rows against the oracle's own formula x + member_deviations(x) @ A
  (enkf.py:192) evaluated on the host with the A each path produced;
* zero-spread rows (constant across members) come out unchanged to rounding: the
  row-local form of test_enkf.py:208-213 (that test's exact identity holds for a wholly
  zero-spread ensemble, T = I, and is pinned bit for bit in test_gpu_parity.py; row by
  row, x + s @ A is exact only where the row mean is, in the reference as here);
* two runs of the product path agree bit for bit (fixed reduction order).
"""

import ctypes

import numpy as np
import pytest

import oracle
from paper_1302_3876_b200 import _native
from paper_1302_3876_b200 import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_1302_3876_b200.build import build
    build()
    import torch
    assert torch.cuda.is_available()


def test_config5_full_size_properties(monkeypatch):
    import torch
    dev = torch.device("cuda", 0)
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info(dev)
    if free < (150 << 30):
        pytest.skip(f"config 5 at full size needs ~150 GB of device memory, {free >> 30} GB free")
    lib = _native.lib()
    s = torch.cuda.current_stream(dev).cuda_stream
    p = W.device_problem_shard(5, 1, 0, dev, 0)
    x, y, r, idx = p["x"], p["perturbed"], p["r"], p["idx"]
    ns, n = x.shape
    nobs = y.shape[0]
    assert (ns, nobs, n) == (1 << 26, 1 << 23, 128)
    zr = torch.arange(3, ns, 65537, device=dev)        # zero-spread rows
    x[zr] = x[zr, :1].repeat(1, n)
    x_zero = x[zr].clone()
    samp = torch.arange(11, ns, 4093, device=dev)      # ~16K sampled rows
    samp = torch.cat([samp, zr])
    x_samp = x[samp].cpu().numpy()
    out = torch.empty_like(x)

    res = {}
    for mode in ("i8", "fp64", "i8-again"):
        if mode == "fp64":
            monkeypatch.setenv("ENKF_GRAM", "fp64")
            monkeypatch.setenv("ENKF_ANOMALY", "fp64")
        plan = _native.Plan(ns, nobs, n, 0)
        monkeypatch.delenv("ENKF_GRAM", raising=False)
        monkeypatch.delenv("ENKF_ANOMALY", raising=False)
        st = _native.EnkfStatus()
        rc = lib.enkf_analysis_f64(plan.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(),
                                   out.data_ptr(), s, ctypes.byref(st))
        assert rc == 0, st.message
        gram = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)
        a = torch.empty((n, n), dtype=torch.float64, device=dev)
        t = torch.empty_like(a)
        assert lib.enkf_plan_reset_status(plan.handle, s) == 0
        assert lib.enkf_ism_gram_f64(plan.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(),
                                     gram.data_ptr(), s) == 0
        assert lib.enkf_ism_levels_f64(plan.handle, gram.data_ptr(), a.data_ptr(), t.data_ptr(), None, s) == 0
        assert lib.enkf_plan_sync_status(plan.handle, s, ctypes.byref(st)) == 0, st.message
        rowsum = out.sum(dim=1)  # a non-finite entry makes its row sum non-finite
        scale = max(float(c.abs().max()) for c in out.split(1 << 21))  # 2 GiB temporaries
        res[mode] = {"gram": gram.cpu().numpy(), "A": a.cpu().numpy(), "samp": out[samp].cpu().numpy(),
                     "rowsum": rowsum,
                     "zero_dev": float(((out[zr] - x_zero).abs() / x_zero.abs().clamp_min(1e-300)).max()),
                     "finite": bool(torch.isfinite(rowsum).all()), "scale": scale}
        del plan
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()

    i8, f64 = res["i8"], res["fp64"]
    got = {}
    for m in ("i8", "fp64"):
        assert res[m]["finite"], m
        # the anomaly update at full size against the oracle's formula with this path's A
        ref = x_samp + oracle.member_deviations(x_samp) @ res[m]["A"]
        got[m + "_vs_oracle_formula"] = np.abs(res[m]["samp"] - ref).max() / res[m]["scale"]
        got[m + "_zero_spread_dev"] = res[m]["zero_dev"]
    # the two kernel families
    got["gram_i8_vs_fp64"] = np.abs(i8["gram"] - f64["gram"]).max() / np.abs(f64["gram"]).max()
    got["A_i8_vs_fp64"] = np.abs(i8["A"] - f64["A"]).max() / np.abs(f64["A"]).max()
    got["xa_rows_i8_vs_fp64"] = np.abs(i8["samp"] - f64["samp"]).max() / f64["scale"]
    got["xa_rowsum_i8_vs_fp64"] = float((i8["rowsum"] - f64["rowsum"]).abs().max()) / (n * f64["scale"])
    print("config5 full-size parity:", {k: float(f"{v:.3g}") for k, v in got.items()})
    for m in ("i8", "fp64"):
        assert got[m + "_vs_oracle_formula"] <= 1e-12, m
        assert got[m + "_zero_spread_dev"] <= 1e-12, m
    assert got["gram_i8_vs_fp64"] <= 1e-13
    assert got["A_i8_vs_fp64"] <= 1e-9
    assert got["xa_rows_i8_vs_fp64"] <= 1e-9
    assert got["xa_rowsum_i8_vs_fp64"] <= 1e-9
    # run-to-run determinism of the product path
    assert torch.equal(i8["rowsum"], res["i8-again"]["rowsum"])
    assert np.array_equal(i8["samp"], res["i8-again"]["samp"])
