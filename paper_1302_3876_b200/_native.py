"""ctypes binding of libenkf_b200.so (the C ABI declared in include/enkf_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device is
visible, every compute entry point raises.  Build the library with
`python -c "import __graft_entry__ as g; g.build()"` (or `python -m
paper_1302_3876_b200.build`).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# ENKF_LIB_VARIANT=<name> loads libenkf_b200_<name>.so (in-tree kernel variants
# built by tools/build_variant.py for A/B timing); the default is the product build.
_VARIANT = os.environ.get("ENKF_LIB_VARIANT", "")
LIB_PATH = os.path.join(_HERE, f"libenkf_b200_{_VARIANT}.so" if _VARIANT else "libenkf_b200.so")

ENKF_OK = 0
ENKF_INVALID_ARGUMENT = 1
ENKF_INDEX_RANGE = 2
ENKF_SINGULAR_UPDATE = 3
ENKF_NOT_SUPPORTED = 4
ENKF_CUDA_ERROR = 5
ENKF_DIVERGED = 6


class EnkfStatus(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int32),
        ("level", ctypes.c_int32),
        ("denominator", ctypes.c_double),
        ("message", ctypes.c_char * 256),
    ]


class EnkfPlanOptions(ctypes.Structure):
    """enkf_plan_options (include/enkf_b200.h): kernel and host-path choices of a plan."""
    _fields_ = [
        ("struct_size", ctypes.c_int32),
        ("gram_kernel", ctypes.c_int32),      # 0 int8-digit tcgen05, 1 FP64 DMMA
        ("anomaly_kernel", ctypes.c_int32),   # 0 int8-digit tcgen05, 1 FP64 DMMA
        ("levels_kernel", ctypes.c_int32),    # 0 cluster, 1 single CTA, 2 level by level
        ("localized_dmma", ctypes.c_int32),
        ("tiny_kernel", ctypes.c_int32),
        ("host_stream", ctypes.c_int32),
        ("host_trace", ctypes.c_int32),
        ("host_chunk_bytes", ctypes.c_int64),
        ("host_ring_bytes", ctypes.c_int64),
        ("host_stream_min_bytes", ctypes.c_int64),
    ]


_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_st = ctypes.POINTER(EnkfStatus)
_opt = ctypes.POINTER(EnkfPlanOptions)

# name -> (restype, argtypes); must match include/enkf_b200.h exactly.
PROTOTYPES = {
    "enkf_version": (ctypes.c_char_p, []),
    "enkf_max_ens": (_i32, []),
    "enkf_set_device": (_i32, [_i32]),
    "enkf_get_device": (_i32, [ctypes.POINTER(_i32)]),
    "enkf_plan_reset_status": (_i32, [_vp, _vp]),
    "enkf_plan_create": (_i32, [_i64, _i64, _i64, ctypes.POINTER(_vp), _st]),
    "enkf_plan_options_default": (_i32, [_opt]),
    "enkf_plan_create_ex": (_i32, [_i64, _i64, _i64, _opt, ctypes.POINTER(_vp), _st]),
    "enkf_plan_destroy": (None, [_vp]),
    "enkf_analysis_f64": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _st]),
    "enkf_analysis_async_f64": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "enkf_plan_sync_status": (_i32, [_vp, _vp, _st]),
    "enkf_analysis_host_f64": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _st]),
    "enkf_ism_gram_f64": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "enkf_ism_levels_f64": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "enkf_anomaly_update_f64": (_i32, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "enkf_ism_solve_f64": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _st]),
    "enkf_member_deviations_f64": (_i32, [_vp, _vp, _i64, _i64, _vp]),
    "enkf_innovations_f64": (_i32, [_vp, _vp, _vp, _vp, _i64, _i64, _vp]),
    "enkf_analysis_localized_f64": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _st]),
    "enkf_analysis_localized_cyclic_f64": (_i32, [_vp, _vp, _vp, _vp, _vp, ctypes.c_double, _vp, _vp, _st]),
    "enkf_forecast_l96_f64": (_i32, [_vp, _vp, _vp, ctypes.c_double, ctypes.c_double, _i32, _vp, _st]),
    "enkf_cycle_l96_f64": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_double, _vp, _vp, _vp, _st, ctypes.POINTER(_i32)]),
    "enkf_cycle_l96_localized_f64": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, ctypes.c_double, ctypes.c_double,
                                            ctypes.c_double, ctypes.c_double, _vp, _vp, _vp, _st,
                                            ctypes.POINTER(_i32)]),
    "enkf_inflate_f64": (_i32, [_vp, _vp, _i64, _i64, ctypes.c_double, _vp]),
    "enkf_comm_unique_id": (_i32, [_vp, _st]),
    "enkf_comm_init": (_i32, [_vp, _i32, _i32, _i32, ctypes.POINTER(_vp), _st]),
    "enkf_comm_destroy": (_i32, [_vp]),
    "enkf_plan_set_comm": (_i32, [_vp, _vp, _st]),
}

_lib = None
_lock = threading.Lock()


class NativeLibraryMissing(RuntimeError):
    """libenkf_b200.so is not built (or failed to load); there is no fallback."""


def lib():
    """Load (once) and return the ctypes handle with typed prototypes."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not found: build it with __graft_entry__.build() "
                    "(the EnKF path has no CPU fallback)")
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in PROTOTYPES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def version() -> str:
    return lib().enkf_version().decode()


def max_ens() -> int:
    return int(lib().enkf_max_ens())


def raise_for_status(code: int, status: EnkfStatus | None, what: str = "") -> None:
    """Map C-ABI status codes onto the reference's exception types
    (errors.py:15-29, enkf.py:54-58, sherman.py:85-108)."""
    if code == ENKF_OK:
        return
    from .errors import SingularUpdateError

    msg = status.message.decode(errors="replace") if status is not None else what
    if code == ENKF_INVALID_ARGUMENT:
        raise ValueError(msg)
    if code == ENKF_INDEX_RANGE:
        raise IndexError(msg)
    if code == ENKF_SINGULAR_UPDATE:
        raise SingularUpdateError(int(status.level), float(status.denominator))
    if code == ENKF_NOT_SUPPORTED:
        raise NotImplementedError(msg)
    if code == ENKF_DIVERGED:
        from .errors import DivergenceError
        raise DivergenceError("state became non-finite", member=int(status.level))
    raise RuntimeError(f"CUDA error in {what}: {msg}")


class on_device:
    """Run the enclosed native calls with `index` as the thread's current CUDA
    device and restore the caller's device afterwards (torch keeps its own)."""

    def __init__(self, index: int):
        self.index = int(index)
        self.prev = None

    def __enter__(self):
        prev = _i32(-1)
        if lib().enkf_get_device(ctypes.byref(prev)) == ENKF_OK:
            self.prev = prev.value
        if lib().enkf_set_device(self.index) != ENKF_OK:
            raise RuntimeError(f"enkf_set_device({self.index}) failed")
        return self

    def __exit__(self, *exc):
        if self.prev is not None and self.prev != self.index:
            lib().enkf_set_device(self.prev)
        return False


def default_options() -> EnkfPlanOptions:
    """Product defaults with the ENKF_* environment overrides applied."""
    o = EnkfPlanOptions()
    if lib().enkf_plan_options_default(ctypes.byref(o)) != ENKF_OK:
        raise RuntimeError("enkf_plan_options_default failed")
    return o


class Plan:
    """Owns one enkf_plan (device workspace for a fixed shape)."""

    def __init__(self, n_state: int, n_obs: int, n_ens: int, device_index: int = 0, options: dict | None = None):
        """`options`: enkf_plan_options fields to change from the defaults (which
        include the process-wide ENKF_* environment overrides), e.g.
        {"gram_kernel": 1, "anomaly_kernel": 1} for the all-IEEE-FP64 step."""
        self.shape = (int(n_state), int(n_obs), int(n_ens))
        self.device_index = int(device_index)
        self._h = _vp()
        st = EnkfStatus()
        opts = default_options()
        for k, v in (options or {}).items():
            if k not in dict(EnkfPlanOptions._fields_) or k == "struct_size":
                raise ValueError(f"unknown plan option {k!r}")
            setattr(opts, k, int(v))
        self.options = opts
        with on_device(self.device_index):
            code = lib().enkf_plan_create_ex(self.shape[0], self.shape[1], self.shape[2], ctypes.byref(opts),
                                             ctypes.byref(self._h), ctypes.byref(st))
        raise_for_status(code, st, "enkf_plan_create_ex")
        self.lock = threading.Lock()

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.enkf_plan_destroy(h)
            self._h = _vp()


_plans: dict = {}
_plans_lock = threading.Lock()


def get_plan(device_index: int, n_state: int, n_obs: int, n_ens: int) -> Plan:
    key = (device_index, int(n_state), int(n_obs), int(n_ens))
    with _plans_lock:
        plan = _plans.get(key)
        if plan is None:
            plan = Plan(n_state, n_obs, n_ens, device_index)
            if len(_plans) > 16:
                _plans.pop(next(iter(_plans)))
            _plans[key] = plan
        return plan
