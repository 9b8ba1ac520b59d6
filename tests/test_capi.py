"""The C-ABI library loads and exports every symbol include/enkf_b200.h
declares (no GPU needed: only non-CUDA entry points are called)."""

import ctypes
import os
import re

import pytest

from paper_1302_3876_b200 import _native
from paper_1302_3876_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "enkf_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(enkf_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def so():
    build()
    return ctypes.CDLL(_native.LIB_PATH)


def test_header_declares_the_surface():
    names = header_functions()
    for must in ("enkf_analysis_f64", "enkf_analysis_host_f64", "enkf_ism_solve_f64",
                 "enkf_ism_gram_f64", "enkf_ism_levels_f64", "enkf_anomaly_update_f64",
                 "enkf_plan_create", "enkf_plan_destroy", "enkf_analysis_localized_f64",
                 "enkf_analysis_localized_cyclic_f64", "enkf_forecast_l96_f64", "enkf_cycle_l96_f64",
                 "enkf_inflate_f64"):
        assert must in names


def test_every_header_symbol_exported(so):
    for name in header_functions():
        assert hasattr(so, name), name


def test_binding_covers_header():
    assert sorted(_native.PROTOTYPES) == header_functions()


def test_version_and_limits(so):
    assert _native.version().startswith("enkf_b200") and "sm_100a" in _native.version()
    assert _native.max_ens() == 128


def test_sm100a_sass_present():
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump missing")
    build()
    out = subprocess.run([tool, "-lelf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([tool, "-sass", _native.LIB_PATH], capture_output=True, text=True).stdout
    funcs = {}
    for chunk in sass.split("Function : ")[1:]:
        name, body = chunk.split("\n", 1)
        funcs[name.strip()] = body
    # the product kernels of the N = 128 step: 5th-gen tensor-core int8 MMAs
    # (UTCIMMA = tcgen05.mma kind::i8), TMEM loads (LDTM = tcgen05.ld), bulk TMA
    # copies (UBLKCP = cp.async.bulk)
    for kern in ("anomaly_i8_kernel", "gram_i8_mma_ls_kernel"):
        body = [b for n, b in funcs.items() if kern in n]
        assert body, kern
        for op in ("UTCIMMA", "LDTM", "UBLKCP"):
            assert op in body[0], (kern, op)
    # the FP64 kernels (N != 128, ENKF_GRAM/ANOMALY=fp64, levels): DMMA + bulk TMA
    for kern in ("gram128_kernel", "rowgemm_ws_kernel", "ism_levels_blocked_kernel"):
        body = [b for n, b in funcs.items() if kern in n]
        assert body and "DMMA.8x8x4" in body[0], kern



def test_plan_options_defaults_and_env_overrides(so, monkeypatch):
    """enkf_plan_options_default: product defaults (int8-digit Gram and anomaly
    kernels, cluster levels, streamed host entry, 256 MiB chunks), with the
    process-wide ENKF_* environment overrides applied on top (no GPU needed)."""
    for k in ("ENKF_GRAM", "ENKF_ANOMALY", "ENKF_LEVELS", "ENKF_HOST_RING_MB", "ENKF_TINY", "ENKF_HOST_STREAM"):
        monkeypatch.delenv(k, raising=False)
    o = _native.default_options()
    assert o.struct_size == ctypes.sizeof(_native.EnkfPlanOptions)
    assert (o.gram_kernel, o.anomaly_kernel, o.levels_kernel) == (0, 0, 0)
    assert (o.localized_dmma, o.tiny_kernel, o.host_stream, o.host_trace) == (1, 1, 1, 0)
    assert o.host_chunk_bytes == 256 << 20 and o.host_ring_bytes == 256 << 20
    assert o.host_stream_min_bytes == 1 << 30
    monkeypatch.setenv("ENKF_GRAM", "fp64")
    monkeypatch.setenv("ENKF_ANOMALY", "fp64")
    monkeypatch.setenv("ENKF_LEVELS", "single")
    monkeypatch.setenv("ENKF_HOST_RING_MB", "1")
    o = _native.default_options()
    assert (o.gram_kernel, o.anomaly_kernel, o.levels_kernel) == (1, 1, 1)
    assert o.host_ring_bytes == 1 << 20
    assert _native.lib().enkf_plan_options_default(None) == _native.ENKF_INVALID_ARGUMENT


def test_plan_create_ex_rejects_bad_options(so):
    """Argument validation happens before any CUDA call: a struct that did not come
    from enkf_plan_options_default, or an out-of-range kernel choice, is
    ENKF_INVALID_ARGUMENT with a null plan."""
    lib = _native.lib()
    for field, value in (("struct_size", 8), ("gram_kernel", 7), ("levels_kernel", -1), ("host_chunk_bytes", -1)):
        o = _native.default_options()
        setattr(o, field, value)
        h, st = ctypes.c_void_p(), _native.EnkfStatus()
        code = lib.enkf_plan_create_ex(16, 8, 4, ctypes.byref(o), ctypes.byref(h), ctypes.byref(st))
        assert code == _native.ENKF_INVALID_ARGUMENT and not h.value, field
        assert b"enkf_plan_options" in st.message
    with pytest.raises(ValueError):
        _native.Plan(16, 8, 4, 0, options={"no_such_option": 1})
