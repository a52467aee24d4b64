"""B200 backend for ringsim.kernels (the reference's kernel boundary,
pkg/src/ringsim/kernels.py:19-40): same contract as ringsim._kernels_ref --
numpy float64 in, numpy float64 out, new arrays, inputs untouched -- with the
arithmetic done by libtokenring.so's sm_100a kernels (bf16 inputs, fp32
accumulate).  A ringsim maintainer drops this file into ``ringsim/`` as
``_kernels_b200.py`` and adds one branch to ``ringsim/kernels.py``:

    elif _choice == "b200":
        from . import _kernels_b200 as _impl

(INTEGRATION.md section 2).  The library is located through
``TOKENRING_LIB`` (this module's own setting, in the reference's process),
defaulting to the in-tree build of this repository.
"""

import ctypes
import os

import numpy as np
import torch                                   # device memory + streams only

_HERE = os.path.dirname(os.path.abspath(__file__))
_DEFAULT = os.path.join(os.path.dirname(_HERE), "paper_2412_20501_b200", "libtokenring.so")
_lib = ctypes.CDLL(os.environ.get("TOKENRING_LIB", _DEFAULT))
_i64, _i32, _vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
_lib.tr_attention_block.argtypes = [_vp] * 5 + [_i64, _i64, _i32, _i32, _i32, _i64, _i64, _vp]
_lib.tr_attention_block.restype = ctypes.c_int
_lib.tr_merge_state.argtypes = [_vp, _vp, _vp, _i32, _vp, _i64, _i32, _i32, _i64, _i64, _vp, _vp]
_lib.tr_merge_state.restype = ctypes.c_int
_lib.tr_last_error.restype = ctypes.c_char_p

MASK_NONE, MASK_FULL, MASK_CAUSAL = 0, 1, 2
BACKEND_NAME = "b200"
TR_DTYPE_F32 = 0


def _dev(x, dtype):
    return torch.as_tensor(np.ascontiguousarray(x)).to("cuda", dtype).contiguous()


def _ok(rc):
    if rc != 0:
        try:
            from .errors import ConfigError, DimensionError, InputError
        except ImportError:                    # loaded outside the ringsim package
            ConfigError = DimensionError = InputError = ValueError
        msg = _lib.tr_last_error().decode()
        raise {-1: DimensionError, -2: InputError, -3: ConfigError}.get(rc, RuntimeError)(msg)


def attention_block(q, k, v, mask_kind, q_offset, k_offset):
    """ref _kernels_ref.py:34-54 / _kernels.pyx:15-65 on the GPU."""
    tq, h, d = q.shape
    out = torch.empty((tq, h, d), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((h, tq), dtype=torch.float32, device="cuda")
    qd, kd, vd = (_dev(x, torch.bfloat16) for x in (q, k, v))
    s = torch.cuda.current_stream().cuda_stream
    _ok(_lib.tr_attention_block(qd.data_ptr(), kd.data_ptr(), vd.data_ptr(), out.data_ptr(),
                                lse.data_ptr(), tq, k.shape[0], h, d, int(mask_kind),
                                int(q_offset), int(k_offset), s))
    return out.double().cpu().numpy(), lse.double().cpu().numpy()


def merge_state(acc_out, acc_lse, blk_out, blk_lse):
    """ref _kernels_ref.py:66-73 / _kernels.pyx:68-102 on the GPU (in place on
    a device copy, so the caller's arrays are untouched)."""
    t, h, d = acc_out.shape
    ao, al = _dev(acc_out, torch.float32), _dev(acc_lse, torch.float32)
    bo, bl = _dev(blk_out, torch.float32), _dev(blk_lse, torch.float32)
    s = torch.cuda.current_stream().cuda_stream
    _ok(_lib.tr_merge_state(ao.data_ptr(), al.data_ptr(), bo.data_ptr(), TR_DTYPE_F32,
                            bl.data_ptr(), t, h, d, t, t, None, s))
    return ao.double().cpu().numpy(), al.double().cpu().numpy()
