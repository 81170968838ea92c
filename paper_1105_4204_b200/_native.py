"""ctypes binding of the C ABI declared in include/trigbf_b200.h.

This is the reference-side binding a maintainer would add next to
``trigbf/_backend.py``: plain pointers and sizes, no torch types.  Loading
fails loudly (``NativeUnavailableError``) -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DimensionError, NativeUnavailableError, ParameterError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libtrigbf_b200.so")

TBF_OK = 0
TBF_ERR_RANGE = 1
TBF_ERR_PARAM = 2
TBF_ERR_DIM = 3
TBF_ERR_CUDA = 4
TBF_ERR_WORKSPACE = 5

TBF_OPT_PIPELINE = 0
TBF_OPT_BATCHES = 1
TBF_OPT_P2_CHUNKS = 3
TBF_OPT_P1_OCC = 4
TBF_OPT_P1_YCHUNKS = 5
TBF_OPT_P1_FOLD = 6
TBF_OPT_HOST_STRIPS = 7
TBF_OPT_HOST_BANDS = 8
TBF_OPT_P2_ORDER = 9
TBF_OPT_LPT_SPLIT = 11  # bits 1/2: planned y-/x-chunks (device entry); 4/8: also in the host entry
TBF_OPT_ZERO_UNIT = 12  # 1: the zero frequency as a packed 1-plane unit (default 0)
TBF_OPT_P1_CLUSTER = 13  # stripes per pass-1 thread-block cluster (default 1 = none)
TBF_LPT_DEFAULT = 3
TBF_LAYOUT_INFO_N = 14
LAYOUT_INFO_FIELDS = ("batches", "batch_terms", "y_chunks", "y_planned", "y_end0", "y_end1", "y_rows_max",
                      "x_chunks", "x_planned", "x_end0", "x_end1", "x_tiles_equal", "x_order", "tiles")

TBF_SPATIAL_RECURSIVE = 0
TBF_SPATIAL_BOX = 1

# Every symbol the header declares (checked by tests/test_abi.py).
EXPORTS = (
    "tbf_workspace_bytes",
    "tbf_layout_info",
    "tbf_bilateral_trig",
    "tbf_bilateral_trig_host",
    "tbf_bilateral_direct",
    "tbf_bilateral_direct_f64",
    "tbf_trig_partial",
    "tbf_trig_partial_rows",
    "tbf_finalize",
    "tbf_range_check",
    "tbf_recursive_smooth_f64",
    "tbf_box_pass_f64",
    "tbf_last_error",
    "tbf_abi_version",
    "tbf_profile_enable",
    "tbf_profile_kinds",
    "tbf_kernel_name",
    "tbf_profile_collect",
    "tbf_profile_timeline",
    "tbf_set_option",
)
ABI_VERSION = 2


class TbfSpatial(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("radius", ctypes.c_int32),
        ("g1", ctypes.c_double),
        ("a1", ctypes.c_double),
        ("a2", ctypes.c_double),
        ("g2", ctypes.c_double),
        ("b1", ctypes.c_double),
        ("b2", ctypes.c_double),
        ("ext_y", ctypes.c_int32),
        ("ext_x", ctypes.c_int32),
    ]


class TbfTerms(ctypes.Structure):
    _fields_ = [
        ("n_terms", ctypes.c_int32),
        ("nu", ctypes.POINTER(ctypes.c_double)),
        ("weight", ctypes.POINTER(ctypes.c_double)),
        ("dnu", ctypes.c_double),
        ("T", ctypes.c_double),
    ]


_lib = None
_lock = threading.Lock()

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double
_sz = ctypes.c_size_t


def _declare(lib):
    lib.tbf_abi_version.restype = _i32
    lib.tbf_abi_version.argtypes = []
    lib.tbf_last_error.restype = ctypes.c_char_p
    lib.tbf_last_error.argtypes = []
    lib.tbf_workspace_bytes.restype = _sz
    lib.tbf_workspace_bytes.argtypes = [_i32, _i32, _i32, ctypes.POINTER(TbfSpatial), _i32, _i32, _i32]
    lib.tbf_layout_info.restype = ctypes.c_int
    lib.tbf_layout_info.argtypes = [_i32, _i32, _i32, ctypes.POINTER(TbfSpatial), _i32, _i32, _i32, _i32,
                                    ctypes.POINTER(_i32), _i32]
    lib.tbf_bilateral_trig.restype = ctypes.c_int
    lib.tbf_bilateral_trig.argtypes = [
        _vp, _vp, _i32, _i32, _i32, ctypes.POINTER(TbfSpatial), ctypes.POINTER(TbfTerms), _i32,
        _vp, _sz, _vp, _vp,
    ]
    lib.tbf_bilateral_trig_host.restype = ctypes.c_int
    lib.tbf_bilateral_trig_host.argtypes = [
        _vp, _vp, _i32, _i32, _i32, ctypes.POINTER(TbfSpatial), ctypes.POINTER(TbfTerms), _i32,
        _vp, _vp, _sz, _vp, _vp,
    ]
    lib.tbf_bilateral_direct.restype = ctypes.c_int
    lib.tbf_bilateral_direct.argtypes = [
        _vp, _i32, _i32, _i32, _vp, _i64, _vp, _i32, _i32, _f64, _i32, _vp, _vp, _vp,
    ]
    lib.tbf_bilateral_direct_f64.restype = ctypes.c_int
    lib.tbf_bilateral_direct_f64.argtypes = lib.tbf_bilateral_direct.argtypes
    lib.tbf_trig_partial.restype = ctypes.c_int
    lib.tbf_trig_partial.argtypes = [
        _vp, _vp, _vp, _i32, _i32, _i32, ctypes.POINTER(TbfSpatial), ctypes.POINTER(TbfTerms),
        _i32, _i32, _i32, _i32, _vp, _sz, _vp,
    ]
    lib.tbf_trig_partial_rows.restype = ctypes.c_int
    lib.tbf_trig_partial_rows.argtypes = [
        _vp, _vp, _vp, _i32, _i32, _i32, ctypes.POINTER(TbfSpatial), ctypes.POINTER(TbfTerms),
        _i32, _i32, _i32, _i32, _i32, _i32, _vp, _sz, _vp,
    ]
    lib.tbf_finalize.restype = ctypes.c_int
    lib.tbf_finalize.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp, _vp]
    lib.tbf_range_check.restype = ctypes.c_int
    lib.tbf_range_check.argtypes = [_vp, _i64, _f64, _vp, _vp]
    lib.tbf_recursive_smooth_f64.restype = ctypes.c_int
    lib.tbf_recursive_smooth_f64.argtypes = [
        _vp, _vp, _i32, _i32, _f64, _f64, _f64, _f64, _f64, _i32, _vp, _vp,
    ]
    lib.tbf_set_option.restype = ctypes.c_int
    lib.tbf_set_option.argtypes = [_i32, _i64]
    lib.tbf_profile_enable.restype = ctypes.c_int
    lib.tbf_profile_enable.argtypes = [_i32]
    lib.tbf_profile_kinds.restype = _i32
    lib.tbf_profile_kinds.argtypes = []
    lib.tbf_kernel_name.restype = ctypes.c_char_p
    lib.tbf_kernel_name.argtypes = [_i32]
    lib.tbf_profile_timeline.restype = _i32
    lib.tbf_profile_timeline.argtypes = [ctypes.POINTER(_f64), ctypes.POINTER(_f64),
                                         ctypes.POINTER(_i32), _i32]
    lib.tbf_profile_collect.restype = ctypes.c_int
    lib.tbf_profile_collect.argtypes = [ctypes.POINTER(_f64), ctypes.POINTER(ctypes.c_longlong), _i32]
    lib.tbf_box_pass_f64.restype = ctypes.c_int
    lib.tbf_box_pass_f64.argtypes = [_vp, _vp, _i32, _i32, _i32, _vp]


def load(path: str | None = None):
    """Load (once) and return the extension library (``TRIGBF_B200_LIB``
    overrides the in-tree path, e.g. for an experimental build)."""
    global _lib
    path = path or os.environ.get("TRIGBF_B200_LIB") or LIB_PATH
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailableError(
                f"sm_100a extension not built ({path}); run `python -m paper_1105_4204_b200.build`"
            )
        lib = ctypes.CDLL(path)
        _declare(lib)
        ver = lib.tbf_abi_version()
        if ver != ABI_VERSION:
            raise NativeUnavailableError(f"ABI mismatch: library {ver}, binding {ABI_VERSION}")
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map a status code to the reference's exception classes (errors.py:4-24)."""
    if rc == TBF_OK:
        return
    msg = load().tbf_last_error().decode(errors="replace")
    if rc in (TBF_ERR_RANGE, TBF_ERR_PARAM):
        raise ParameterError(msg)
    if rc == TBF_ERR_DIM:
        raise DimensionError(msg)
    raise RuntimeError(f"trigbf_b200 error {rc}: {msg}")


class KernelProfiler:
    """Context manager: per-kernel device time of every launch inside it,
    measured with CUDA events on the launch stream by the library."""

    def __enter__(self):
        lib = load()
        self.lib = lib
        n = lib.tbf_profile_kinds()
        self.n = n
        self.names = [lib.tbf_kernel_name(k).decode() for k in range(n)]
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_longlong * n)()
        lib.tbf_profile_collect(ms, cnt, n)  # drop anything stale
        lib.tbf_profile_enable(1)
        self.result = {}
        return self

    def __exit__(self, *exc):
        self.lib.tbf_profile_enable(0)
        ms = (ctypes.c_double * self.n)()
        cnt = (ctypes.c_longlong * self.n)()
        check(self.lib.tbf_profile_collect(ms, cnt, self.n))
        self.result = {self.names[k]: (float(ms[k]), int(cnt[k])) for k in range(self.n) if cnt[k]}
        return False
