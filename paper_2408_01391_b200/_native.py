"""ctypes binding of the C ABI in include/ftk_b200.h (libftkb200.so).

There is no fallback: if the shared library is missing, or no CUDA device is
present when a compute entry point is called, this module raises.  Build the
library with ``python -c "import __graft_entry__ as g; g.build()"`` (or
``python paper_2408_01391_b200/build.py``).
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FTK_LIB_PATH") or os.path.join(HERE, "_lib", "libftkb200.so")

FTK_OK, FTK_OVERFLOW = 0, 1
FTK_F32, FTK_F64 = 0, 1
VARIANT_AUTO, VARIANT_EXACT, VARIANT_TC = 0, 1, 2
VARIANT_TC_PAIR, VARIANT_TC_NARROW, VARIANT_F64_DMMA, VARIANT_F64_DFMA = 3, 4, 5, 6

_i64, _i32, _p, _dbl, _int = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_double, ctypes.c_int


class Injection(ctypes.Structure):
    _fields_ = [("n", _i64), ("bi", _p), ("bj", _p), ("ei", _p), ("ej", _p), ("bit", _p),
                ("applied", _p), ("before", _p), ("after", _p), ("n_dev", _p)]


class Events(ctypes.Structure):
    _fields_ = [("cap", _i64), ("rec", _p), ("delta", _p), ("count", _p)]


# name -> (restype, argtypes); mirrors include/ftk_b200.h exactly
PROTOTYPES = {
    "ftk_last_error": (ctypes.c_char_p, []),
    "ftk_version": (_int, []),
    "ftk_launch_count": (_i64, []),
    "ftk_add_launches": (None, [_i64]),
    "ftk_ctx_create": (_p, [_int]),
    "ftk_ctx_destroy": (None, [_p]),
    "ftk_row_sq_norms": (_int, [_p, _int, _p, _i64, _i64, _p, _p]),
    "ftk_row_info": (_int, [_p, _p, _i64, _i64, _p, _p]),
    "ftk_kpp_d2": (_int, [_p, _int, _p, _i64, _i64, _i64, _int, _p, _p]),
    "ftk_kpp_update": (_int, [_p, _int, _p, _i64, _i64, _i64, _p, _int, _p, _p, _i64, _p]),
    "ftk_kpp_search": (_int, [_p, _p, _i64, _dbl, _p, _p, _p]),
    "ftk_ctx_set_rows": (_int, [_p, _p, _i64, _i64, _p]),
    "ftk_row_info64": (_int, [_p, _p, _i64, _i64, _p, _p, _p]),
    "ftk_ctx_set_rows64": (_int, [_p, _p, _i64, _i64, _p, _p]),
    "ftk_ctx_generation": (_i64, [_p]),
    "ftk_ctx_set_label_hint": (_int, [_p, _p, _i64]),
    "ftk_ctx_set_option": (_int, [_p, _int, _i64]),
    "ftk_assign": (_int, [_p, _int, _int, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _p, _p,
                          _p, _p]),
    "ftk_checked_assign": (_int, [_p, _int, _int, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64,
                                  _dbl, _dbl, _i64, _p, _p, _p, _p, _p]),
    "ftk_gemm": (_int, [_p, _int, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _dbl, _dbl, _i64,
                        _p, _p, _p, _p]),
    "ftk_update_sums": (_int, [_p, _int, _p, _p, _i64, _i64, _i64, _p, _p, _p, _p, _p]),
    "ftk_dmr_compare": (_int, [_p, _p, _p, _p, _p, _i64, _i64, _p, _p]),
    "ftk_update_finalize": (_int, [_p, _int, _p, _p, _i64, _i64, _p, _p, _p]),
    "ftk_reseed_empty": (_int, [_p, _int, _p, _i64, _i64, _p, _i64, _p, _p, _p]),
    "ftk_sq_dists": (_int, [_p, _int, _p, _p, _i64, _p, _p]),
    "ftk_pairwise_sum": (_int, [_p, _p, _i64, _p, _p]),
    "ftk_movement": (_int, [_p, _int, _p, _p, _i64, _i64, _dbl, _p, _p]),
    "ftk_labels_equal": (_int, [_p, _p, _p, _i64, _p, _p]),
    "ftk_own_sq_dists": (_int, [_p, _int, _p, _p, _p, _i64, _i64, _p, _p]),
    "ftk_flip_f64": (_int, [_p, _p, _i64, _i64, _i64, _i64, _p, _p]),
    "ftk_tc_fallback_rows": (_int, [_p, _p, _p]),
    "ftk_tc_last_kernel_ms": (_int, [_p, _p]),
    "ftk_abft_flags_total": (_int, [_p, _p, _int, _p]),
    "ftk_h2d": (_int, [_p, _p, _p, _i64, _p]),
    "ftk_tc_raw_dots": (_int, [_p, _int, _p, _p, _p, _i64, _i64, _i64, _p, _p, _p, _p]),
}

_LIB = None


def load():
    """Load libftkb200.so (no CUDA call happens at load time)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"CUDA extension not built: {LIB_PATH} is missing. Run "
            "`python paper_2408_01391_b200/build.py` (nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


class FTKError(RuntimeError):
    pass


def check(rc, what=""):
    if rc == FTK_OK or rc == FTK_OVERFLOW:
        return rc
    msg = load().ftk_last_error().decode(errors="replace")
    if rc == -3:
        raise ValueError(f"{what}: unsupported configuration: {msg}")
    raise FTKError(f"{what} failed ({rc}): {msg}")


def launch_count():
    return int(load().ftk_launch_count())
