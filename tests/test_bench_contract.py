"""bench.py keeps the driver's JSON contract (one line on rank 0 with the base keys,
roofline, cpu_baseline, e2e, clocks, gpu_launches) on a shrunk config-5 workload,
and the reference arm prints its line; the CPU part runs everywhere."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--scale-log2", "6"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["value"] > 0 and d["higher_is_better"] is True


@pytest.mark.gpu
def test_bench_line_contract():
    d = _run(["--steps", "3", "--warmup", "3", "--scale-log2", "6", "--e2e-steps", "1"])
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] < 1.2 and r["peak"] > 0 and r["unit"] in ("GB/s", "TFLOP/s")
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert d["gpu_launches"] > 0
    assert d["ism_sweep"] is None or 0 < d["ism_sweep"]["frac"] < 1.2
    assert 0 < d["roofline_step"]["frac"] < 1.2 and d["energy_j_per_step"] is None or d["energy_j_per_step"] > 0
    assert d["strict_fp64"]["value"] > 0 and "IEEE" in d["strict_fp64"]["dtype"]
    assert "emulation" in d["dtype"]
    assert d["overflow_cliff"]["gram_ms_fallback"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_bench_small_configs(cfg):
    """Driver-visible throughput of the latency-bound configs 1-3 (one analysis per step)."""
    d = _run(["--config", str(cfg), "--steps", "20", "--warmup", "3", "--e2e-steps", "3"])
    assert BASE_KEYS <= set(d) and d["value"] > 0 and d["config"]["workload"].startswith(f"config{cfg}")
    assert d["cpu_baseline"]["extrapolated"] is False and d["cpu_baseline"]["value"] > 0
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


def test_gpus_beyond_visible_fails():
    """`--gpus N` with fewer visible GPUs exits non-zero instead of timing one rank."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64", "--steps", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode != 0 and "64" in out.stderr


def test_reference_arm_small_config_not_extrapolated():
    """Configs 1-3 run the oracle on the full configuration: no extrapolation."""
    d = _run(["--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "0"])
    assert d["impl"] == "reference" and d["extrapolated"] is False
    assert d["config"]["workload"].startswith("config1") and d["value"] > 0


def test_reference_arm_flags_extrapolation():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--scale-log2", "8"])
    assert d["extrapolated"] is True and d["measured_seconds_per_sample_step"] > 0
    lin = d["cpu_baseline"]["linearity"]
    assert len(lin["seconds"]) == 2 and all(t > 0 for t in lin["seconds"])


def test_nccl_init_lines_parsing(tmp_path):
    """rank 0 folds the per-rank NCCL communicator-init lines into its JSON line."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    (tmp_path / "nccl.host.1.log").write_text("host:1:1 NCCL INFO Bootstrap\n"
                                              "host:1:1 NCCL INFO ncclCommInitRank comm 0x1 rank 0 nranks 2 - Init COMPLETE\n")
    (tmp_path / "nccl.host.2.log").write_text("host:2:2 NCCL INFO ncclCommInitRank comm 0x2 rank 1 nranks 2 - Init COMPLETE\n")
    lines = bench.nccl_init_lines(str(tmp_path))
    assert len(lines) == 2 and all("nranks 2" in ln for ln in lines)
    assert bench.nccl_init_lines(None) is None
