"""ctypes binding of libtokenring.so (the C ABI declared in include/tokenring.h).

The library is built in-tree (``python -m paper_2412_20501_b200.build``).  There
is no fallback: if the shared object is missing or fails to load, every
compute entry point raises -- the product path never silently degrades to a
CPU or PyTorch implementation.  There is no library-selection switch either:
the product loads ``libtokenring.so`` next to this file (A/B scripts and the
experiments build load their own libraries explicitly, see ``load_library``).
"""

import ctypes
import os
import threading

from .errors import ConfigError, DimensionError, InputError, RingsimError, ScheduleError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtokenring.so")

TR_OK = 0
TR_ERR_DIMENSION = -1
TR_ERR_INPUT = -2
TR_ERR_CONFIG = -3
TR_ERR_CUDA = -4
TR_ERR_UNSUPPORTED = -5
TR_ERR_TIMEOUT = -6

TR_DTYPE_F32 = 0
TR_DTYPE_BF16 = 1
TR_MERGE_MAX = 16

# every symbol include/tokenring.h declares
EXPORTS = ("tr_attention_block", "tr_attention_segments", "tr_attention_segments_push",
           "tr_attention_segments_push_rel",
           "tr_merge_state", "tr_merge_n", "tr_partial_init",
           "tr_splitmix_bf16", "tr_flag_set", "tr_flag_wait", "tr_flag_set_rel",
           "tr_flag_wait_rel", "tr_epoch_add", "tr_copy_async",
           "tr_enable_peer_access", "tr_poll_error", "tr_clear_error",
           "tr_set_flag_timeout_ms", "tr_set_launch_overlap", "tr_version",
           "tr_kernel_count", "tr_kernel_name", "tr_last_error")


class CudaError(RingsimError, RuntimeError):
    """A CUDA runtime/driver call inside libtokenring failed."""


class UnsupportedError(RingsimError, ValueError):
    """The sm_100a kernels do not cover this shape."""


class Segment(ctypes.Structure):
    """tr_segment: local rows [row0, row0+rows) at global positions pos0.."""
    _fields_ = [("row0", ctypes.c_int64), ("rows", ctypes.c_int64), ("pos0", ctypes.c_int64)]


_lib = None
_lock = threading.Lock()


def _declare(lib):
    i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    lib.tr_attention_block.argtypes = [vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, i64, i64, vp]
    lib.tr_attention_segments.argtypes = [vp, vp, vp, vp, vp, i64, i64, i32, i32,
                                          ctypes.POINTER(Segment), i32,
                                          ctypes.POINTER(Segment), i32, i32, i32, vp]
    lib.tr_attention_segments_push.argtypes = [vp, vp, vp, vp, vp, i64, i64, i32, i32,
                                               ctypes.POINTER(Segment), i32,
                                               ctypes.POINTER(Segment), i32, i32, i64, i64,
                                               vp, vp, ctypes.c_uint64, vp]
    try:    # A/B builds older than the epoch-relative ABI lack these four
        lib.tr_attention_segments_push_rel.argtypes = [vp, vp, vp, vp, vp, i64, i64, i32, i32,
                                                       ctypes.POINTER(Segment), i32,
                                                       ctypes.POINTER(Segment), i32, i32, i64,
                                                       i64, vp, vp, vp, i64, vp]
        lib.tr_flag_set_rel.argtypes = [vp, vp, i64, vp]
        lib.tr_flag_wait_rel.argtypes = [vp, vp, i64, vp]
        lib.tr_epoch_add.argtypes = [vp, i64, vp]
        for name in ("tr_attention_segments_push_rel", "tr_flag_set_rel", "tr_flag_wait_rel",
                     "tr_epoch_add"):
            getattr(lib, name).restype = ctypes.c_int
    except AttributeError:
        pass
    lib.tr_merge_state.argtypes = [vp, vp, vp, i32, vp, i64, i32, i32, i64, i64, vp, vp]
    lib.tr_merge_n.argtypes = [vp, vp, i64, ctypes.POINTER(vp), i32, ctypes.POINTER(vp),
                               ctypes.POINTER(i64), i32, i64, i32, i32, vp, vp]
    lib.tr_partial_init.argtypes = [vp, vp, i64, i32, i32, vp]
    lib.tr_splitmix_bf16.argtypes = [ctypes.c_uint64, i64, i64, ctypes.c_double,
                                     ctypes.c_double, vp, vp]
    lib.tr_flag_set.argtypes = [vp, ctypes.c_uint64, vp]
    lib.tr_flag_wait.argtypes = [vp, ctypes.c_uint64, vp]
    lib.tr_copy_async.argtypes = [vp, vp, ctypes.c_uint64, vp]
    lib.tr_enable_peer_access.argtypes = [i32]
    lib.tr_poll_error.argtypes = []
    lib.tr_clear_error.argtypes = []
    lib.tr_clear_error.restype = None
    lib.tr_set_flag_timeout_ms.argtypes = [ctypes.c_uint64]
    lib.tr_set_flag_timeout_ms.restype = None
    if hasattr(lib, "tr_set_launch_overlap"):   # absent from older A/B builds
        lib.tr_set_launch_overlap.argtypes = [i32]
        lib.tr_set_launch_overlap.restype = i32
    for name in ("tr_attention_block", "tr_attention_segments", "tr_attention_segments_push",
                 "tr_merge_state", "tr_merge_n",
                 "tr_partial_init", "tr_splitmix_bf16", "tr_flag_set", "tr_flag_wait",
                 "tr_copy_async", "tr_enable_peer_access", "tr_poll_error"):
        getattr(lib, name).restype = ctypes.c_int
    lib.tr_version.restype = ctypes.c_char_p
    lib.tr_version.argtypes = []
    lib.tr_kernel_count.restype = ctypes.c_int32
    lib.tr_kernel_count.argtypes = []
    lib.tr_kernel_name.restype = ctypes.c_char_p
    lib.tr_kernel_name.argtypes = [i32]
    lib.tr_last_error.restype = ctypes.c_char_p
    lib.tr_last_error.argtypes = []


def load_library(path):
    """ctypes handle of a libtokenring build at ``path`` with the C ABI declared."""
    if not os.path.exists(path):
        raise ImportError(f"{path} is not built; run `python -m paper_2412_20501_b200.build` "
                          "(there is no CPU fallback)")
    handle = ctypes.CDLL(path)
    _declare(handle)
    return handle


def lib():
    """Load (once) and return the product library; raises if it is not built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                _lib = load_library(LIB_PATH)
    return _lib


def use_library(path):
    """Point this process at another build of the library (A/B scripts and the
    experiments build only -- never the product path).  Call before any
    compute call."""
    global _lib
    with _lock:
        _lib = load_library(path)
    return _lib


def check(status):
    """Map a TR_* status onto the reference's exception taxonomy (errors.py:4-25)."""
    if status == TR_OK:
        return
    msg = lib().tr_last_error().decode(errors="replace")
    if status == TR_ERR_DIMENSION:
        raise DimensionError(msg)
    if status == TR_ERR_INPUT:
        raise InputError(msg)
    if status == TR_ERR_CONFIG:
        raise ConfigError(msg)
    if status == TR_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    if status == TR_ERR_TIMEOUT:
        raise ScheduleError(msg)
    raise CudaError(msg)
