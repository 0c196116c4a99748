"""ctypes binding of ``libmk_strassen.so`` (the C ABI declared in include/mk_strassen.h).

The shared library is the only compute path of this package: there is no CPU or
PyTorch fallback. Importing the package works without a GPU (so CPU-only tooling and
tests can inspect the ABI), but every compute call raises ``EngineUnavailable`` when
the library is missing or no CUDA device is present.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .core import AliasError, DimensionError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmk_strassen.so")

# status codes (include/mk_strassen.h)
MK_OK, MK_ERR_DIMENSION, MK_ERR_ALIAS, MK_ERR_CUDA, MK_ERR_WORKSPACE, MK_ERR_ARG, MK_ERR_INEXACT = range(7)

# algorithm ids (include/mk_strassen.h enum mk_algo)
ALGO_IDS = {
    "naive": 0,
    "strassen": 1,
    "winograd-block": 2,
    "winograd-knuth": 3,
    "winograd-knuth-8call": 4,
    "two-temp": 5,
    "in-place": 6,
}
MK_OPT_FUSE_PREADDS = 1
MK_OPT_PLAN = 2  # 0 breadth-first (default), 1 depth-first (workspace-minimal), 2 hybrid
MK_OPT_LITERAL_TAIL = 3  # two-temp: 0 literal to the leaves (default), 1 breadth-first last two levels
MK_OPT_LEAF_SLICES = 4  # 0 DMMA leaves (default), 4..8 INT8 tensor-core (Ozaki) leaves with that many slices
MK_OPT_LEAF_MIN_LOG2 = 5  # INT8 leaves only for products with m*n*k >= 2^v (default 29)
MK_OPT_BFS_GROUP = 6  # top-level products per breadth-first pass (0 = auto)
MK_OPT_PDL = 9  # sub-wave leaf launches / small additions as programmatic dependent launches: 1 (default), 0 plain
MK_OPT_PIPELINE = 10  # pipelined breadth-first plan: 0 never, 1 auto (default: leaves long enough to hide transforms), 2 every narrow-leaf call
MK_OPT_HOST_GROUP = 8  # host path, 2 levels: middle products as one grouped pass (-1 auto, 0 off, k: after k products)
MK_OPT_LITERAL_STREAMS = 7  # two-temp / in-place: 1 additions off the critical path on side streams (default), 0 one stream

# every exported symbol with (restype, argtypes)
_I64, _VP, _INT, _SZ, _DP = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(ctypes.c_double)
SIGNATURES = {
    "mk_version": (_INT, []),
    "mk_launch_count": (ctypes.c_longlong, []),
    "mk_timing_begin": (_INT, []),
    "mk_timing_end": (_INT, [_DP, ctypes.POINTER(_INT), _DP]),
    "mk_fp64_peak": (_INT, [_DP, _VP]),
    "mk_set_option": (_INT, [_INT, _INT]),
    "mk_get_option": (_INT, [_INT, ctypes.POINTER(ctypes.c_int)]),
    "mk_set_thread_option": (_INT, [_INT, _INT]),
    "mk_last_error": (ctypes.c_char_p, []),
    "mk_dgemm": (_INT, [_VP, _I64, _VP, _I64, _VP, _I64, _I64, _I64, _I64, _VP]),
    "mk_ozaki_workspace_bytes": (_SZ, [_I64, _I64, _I64, _INT]),
    "mk_ozaki_dgemm": (_INT, [_VP, _I64, _VP, _I64, _VP, _I64, _I64, _I64, _I64, _INT, _VP, _SZ, _VP]),
    "mk_levels_for_policy": (_INT, [_I64, _INT, _I64, _INT, ctypes.POINTER(_INT)]),
    "mk_workspace_bytes": (_SZ, [_INT, _I64, _INT]),
    "mk_strassen": (_INT, [_INT, _VP, _I64, _VP, _I64, _VP, _I64, _I64, _INT, _VP, _SZ, _VP]),
    "mk_rect_workspace_bytes": (_SZ, [_INT, _I64, _I64, _I64, _INT]),
    "mk_multiply_rect": (_INT, [_INT, _VP, _I64, _VP, _I64, _VP, _I64, _I64, _I64, _I64, _INT, _VP, _SZ, _VP]),
    "mk_block_combine": (_INT, [_VP, _I64, ctypes.POINTER(_VP), ctypes.POINTER(_I64), _DP, _INT, _I64, _I64, _VP]),
    "mk_i64_to_f64": (_INT, [_VP, _I64, _VP, _I64, _I64, _I64, _VP]),
    "mk_f64_to_i64": (_INT, [_VP, _I64, _VP, _I64, _I64, _I64, _VP]),
    "mk_absmax_f64": (_INT, [_VP, _I64, _I64, _I64, _DP, _VP]),
    "mk_absmax_i64": (_INT, [_VP, _I64, _I64, _I64, _DP, _VP]),
    "mk_product_count": (_INT, [_INT, _INT]),
    "mk_partial_workspace_bytes": (_SZ, [_INT, _I64, _INT]),
    "mk_host_workspace_bytes": (_SZ, [_INT, _I64, _INT]),
    "mk_copy_to_device": (_INT, [_VP, _I64, _VP, _I64, _I64, _I64, _VP]),
    "mk_copy_to_host": (_INT, [_VP, _I64, _VP, _I64, _I64, _I64, _VP]),
    "mk_strassen_host": (_INT, [_INT, _VP, _I64, _VP, _I64, _VP, _I64, _I64, _INT, _VP, _VP, _VP, _I64, _VP, _SZ,
                                _VP, _VP]),
    "mk_enable_peer_access": (_INT, [_INT]),
    "mk_rect_partial_workspace_bytes": (_SZ, [_INT, _I64, _I64, _I64, _INT, _INT]),
    "mk_multiply_rect_partial": (_INT, [_INT, _VP, _I64, _VP, _I64, _VP, _I64, _I64, _I64, _I64, _INT, _INT, _INT,
                                        _INT, _VP, _SZ, _VP]),
    "mk_strassen_partial_slabs": (_INT, [_INT, _VP, _I64, _VP, _I64, ctypes.POINTER(_VP), _INT, _I64, _I64, _I64,
                                         _INT, _INT, _INT, _INT, _VP, _SZ, _VP]),
    "mk_overlap_order": (_INT, [_INT, ctypes.POINTER(_INT), ctypes.POINTER(_INT)]),
    "mk_strassen_partial": (_INT, [_INT, _VP, _I64, _VP, _I64, _VP, _I64, _I64, _INT, _INT, _INT, _INT, _VP, _SZ,
                                   _VP]),
    "mk_multi_gpu_workspace_bytes": (_SZ, [_INT, _I64, _INT, _INT, _INT]),
    "mk_multi_gpu_winograd": (_INT, [_INT, _INT, ctypes.POINTER(_INT), _VP, _I64, _VP, _I64, _VP, _I64, _I64, _INT,
                                     ctypes.POINTER(_VP), ctypes.POINTER(_SZ), ctypes.POINTER(_VP)]),
}


class EngineUnavailable(RuntimeError):
    """The sm_100a engine cannot run here (library not built, or no CUDA device)."""


class EngineError(RuntimeError):
    """A CUDA-level failure inside the engine."""


class ExactnessError(ValueError):
    """Integer operands whose product cannot be formed exactly in FP64 on the engine."""


_lock = threading.Lock()
_lib = None


def load(required: bool = True):
    """Load (once) and return the ctypes library; raise EngineUnavailable if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                if required:
                    raise EngineUnavailable(
                        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                    )
                return None
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return sorted(SIGNATURES)


def check(rc: int, what: str) -> None:
    """Map an engine status code to the reference's exception types."""
    if rc == MK_OK:
        return
    msg = f"{what}: {load().mk_last_error().decode(errors='replace')}"
    if rc == MK_ERR_DIMENSION:
        raise DimensionError(msg)
    if rc == MK_ERR_ALIAS:
        raise AliasError(msg)
    if rc == MK_ERR_INEXACT:
        raise ExactnessError(msg)
    if rc in (MK_ERR_ARG, MK_ERR_WORKSPACE):
        raise ValueError(msg)
    raise EngineError(msg)
