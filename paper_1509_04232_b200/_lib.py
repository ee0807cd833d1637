"""ctypes binding of libspx.so (the C ABI declared in include/spx.h).

The library is the only compute path: if it cannot be loaded, every kernel
call raises -- there is no CPU fallback.
"""

import ctypes
import os

from .errors import DimensionMismatchError, InvalidSettingsError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libspx.so")
# Development only: A/B kernel variants built by tools/build_variants.py.
LIB_PATH = os.environ.get("SPX_LIB_VARIANT", LIB_PATH)

SPX_OK = 0
SPX_ERR_INVALID_SETTINGS = 1
SPX_ERR_DIMENSION = 2
SPX_ERR_CUDA = 3
SPX_ERR_NOMEM = 4
SPX_ERR_VALUE = 5

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
D = ctypes.c_double


class SpxSettings(ctypes.Structure):
    _fields_ = [
        ("width", I64), ("height", I64), ("s", I64), ("ns_r", I64), ("ns_c", I64),
        ("compactness", D), ("no_iters", I32), ("color_space", I32), ("connectivity", I32),
        ("perturb", I32), ("tile_len", I64), ("min_size", I64), ("early_stop", D),
    ]


class SpxTiming(ctypes.Structure):
    _fields_ = [
        ("convert", ctypes.c_float), ("init", ctypes.c_float), ("perturb", ctypes.c_float),
        ("connectivity", ctypes.c_float), ("total", ctypes.c_float),
        ("associate", ctypes.c_float * 1024), ("update", ctypes.c_float * 1024),
        ("n_associate", I32), ("n_update", I32),
    ]


# name -> (restype, argtypes); must match include/spx.h
SIGNATURES = {
    "spx_last_error": (ctypes.c_char_p, []),
    "spx_name": (ctypes.c_char_p, []),
    "spx_abi_version": (I32, []),
    "spx_debug_tables": (I32, [P, P, P]),
    "spx_debug_sqrt_error": (I32, [P]),
    "spx_debug_ddiv_check": (I32, [I64, ctypes.c_uint64, P]),
    "spx_convert_band": (I32, [P, P, I64, I64, I32, I64, I64, P]),
    "spx_init_centers_range": (I32, [P, I64, I64, I64, I64, P, P, I64, I64, P]),
    "spx_perturb_range": (I32, [P, I64, I64, P, P, I64, I64, P]),
    "spx_associate_band": (I32, [P, I64, I64, P, P, I64, P, I64, I64, I64, D, I64, I64, P]),
    "spx_accumulate_range": (I32, [P, P, I64, I64, P, I64, I64, I64, I64, I64, I64, P]),
    "spx_accumulate_spill": (I32, [P, P, I64, I64, P, I64, I64, I64, I64, P, P]),
    "spx_reduce_range": (I32, [P, I64, P, P, P, P, P, I64, I64, P]),
    "spx_weak_band": (I32, [P, P, I64, I64, I64, I64, P]),
    "spx_strict_fill": (I32, [P, P, I64, I64, I64, P]),
    "spx_center_shift": (I32, [P, P, I64, P, P]),
    "spx_pairwise_sum": (I32, [P, I64, P, P]),
    "spx_engine_create": (I32, [ctypes.POINTER(SpxSettings), I64, I32, ctypes.POINTER(P)]),
    "spx_engine_destroy": (I32, [P]),
    "spx_engine_segment": (I32, [P, P, I64, P, P, P, P, P, P]),
    "spx_engine_segment_host": (I32, [P, P, I64, P, P, P, P, P]),
    "spx_engine_submit_host": (I32, [P, P, I64, P, P, P, P, P]),
    "spx_engine_wait": (I32, [P]),
    "spx_engine_ticket": (I64, [P]),
    "spx_engine_wait_ticket": (I32, [P, I64]),
    "spx_engine_ticket_time": (I32, [P, I64, ctypes.POINTER(ctypes.c_float)]),
    "spx_engine_output_layout": (I32, [P, I64, P]),
    "spx_engine_set_host_chunk": (I32, [P, I64]),
    "spx_engine_set_lanes": (I32, [P, I32]),
    "spx_engine_last_lanes": (I32, [P]),
    "spx_engine_timing": (I32, [P, ctypes.POINTER(SpxTiming)]),
    "spx_engine_last_launches": (I64, [P]),
    "spx_engine_fused_path": (I32, [P]),
    "spx_strip_create": (I32, [ctypes.POINTER(SpxSettings), I64, I64, I32, ctypes.POINTER(P)]),
    "spx_strip_destroy": (I32, [P]),
    "spx_strip_geometry": (I32, [P, P]),
    "spx_strip_begin": (I32, [P, P, P]),
    "spx_strip_associate": (I32, [P, I32, P]),
    "spx_strip_update": (I32, [P, P]),
    "spx_strip_associate_part": (I32, [P, I32, I32, P]),
    "spx_strip_update_part": (I32, [P, I32, P]),
    "spx_strip_shift_local": (I32, [P, P, P]),
    "spx_strip_pack_centres": (I32, [P, P, P, P]),
    "spx_strip_unpack_centres": (I32, [P, P, P, P]),
    "spx_strip_pack_sums": (I32, [P, P, P, P]),
    "spx_strip_unpack_sums": (I32, [P, P, P, P]),
    "spx_strip_pack_labels": (I32, [P, P, P, P]),
    "spx_strip_unpack_labels": (I32, [P, P, P, P]),
    "spx_strip_finish": (I32, [P, P, P, P, P, P]),
}

_lib = None


class SpxCudaError(RuntimeError):
    """A CUDA failure inside libspx (no CPU fallback exists)."""


def load():
    """Load libspx.so; raises ImportError when it is missing or unloadable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libspx.so not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc, what=""):
    if rc == SPX_OK:
        return
    msg = (load().spx_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == SPX_ERR_INVALID_SETTINGS:
        raise InvalidSettingsError(text)
    if rc == SPX_ERR_DIMENSION:
        raise DimensionMismatchError(text)
    if rc == SPX_ERR_NOMEM:
        raise MemoryError(text)
    if rc == SPX_ERR_VALUE:
        raise ValueError(text)
    raise SpxCudaError(text)
