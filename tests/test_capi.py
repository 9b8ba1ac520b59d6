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

