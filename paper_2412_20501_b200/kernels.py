"""Kernel boundary: the two primitives of ``ringsim.kernels``
(``pkg/src/ringsim/kernels.py:33-40``) on CUDA tensors, executed by the
sm_100a kernels of libtokenring.so through its C ABI.

``attention_block(q, k, v, mask_kind, q_offset, k_offset) -> (out, lse)``
    q (Tq,H,D), k/v (Tk,H,D) bf16 CUDA tensors -> out (Tq,H,D) bf16,
    lse (H,Tq) float32 (ref ``_kernels_ref.py:34-54``).
``merge_state(acc_out, acc_lse, blk_out, blk_lse) -> (out, lse)``
    returns a new float32 accumulator (ref ``_kernels_ref.py:66-73``);
    ``merge_state_`` is the in-place form the executors use.

Unlike the reference there is exactly one backend: ``BACKEND`` names it and
there is no environment switch and no CPU fallback.
"""

import ctypes

import torch

from . import _lib
from .errors import DimensionError

MASK_NONE = 0
MASK_FULL = 1
MASK_CAUSAL = 2

BACKEND = "cuda-sm100a"

# Number of device kernels this process has launched through libtokenring
# (bench.py reports the count inside its timed region as ``gpu_launches``).
LAUNCHES = 0


def _count(n):
    global LAUNCHES
    LAUNCHES += n


def _stream(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _on(t):
    """Make ``t``'s device current for a C-ABI call: the library launches on
    the calling thread's current device (and sets per-device kernel
    attributes there), so a process driving several GPUs must switch."""
    return torch.cuda.device(t.device)


def _require_cuda(name, t, dtype=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise DimensionError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise DimensionError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise DimensionError(f"{name} must be contiguous")


def _check_qkv(q, k, v):
    for n, t in (("q", q), ("k", k), ("v", v)):
        _require_cuda(n, t, torch.bfloat16)
        if t.dim() != 3:
            raise DimensionError(f"{n} must have shape (T, H, D), got {tuple(t.shape)}")
    if q.shape[1] != k.shape[1] or q.shape[1] != v.shape[1]:
        raise DimensionError(f"head counts differ: q={q.shape[1]} k={k.shape[1]} v={v.shape[1]}")
    if q.shape[2] != k.shape[2] or q.shape[2] != v.shape[2]:
        raise DimensionError(f"head dims differ: q={q.shape[2]} k={k.shape[2]} v={v.shape[2]}")
    if k.shape[0] != v.shape[0]:
        raise DimensionError(f"k has {k.shape[0]} tokens but v has {v.shape[0]}")


def attention_block(q, k, v, mask_kind=MASK_NONE, q_offset=0, k_offset=0, out=None, lse=None):
    _check_qkv(q, k, v)
    tq, h, d = q.shape
    tk = k.shape[0]
    if out is None:
        out = torch.empty((tq, h, d), dtype=torch.bfloat16, device=q.device)
    if lse is None:
        lse = torch.empty((h, tq), dtype=torch.float32, device=q.device)
    _require_cuda("out", out, torch.bfloat16)
    _require_cuda("lse", lse, torch.float32)
    if tuple(out.shape) != (tq, h, d) or tuple(lse.shape) != (h, tq):
        raise DimensionError(f"out must be {(tq, h, d)} and lse {(h, tq)}, got "
                             f"{tuple(out.shape)} / {tuple(lse.shape)}")
    for n, t in (("k", k), ("v", v), ("out", out), ("lse", lse)):
        if t.device != q.device:
            raise DimensionError(f"{n} is on {t.device}, q on {q.device}")
    with _on(q):
        _lib.check(_lib.lib().tr_attention_block(
            _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), tq, tk, h, d, int(mask_kind),
            int(q_offset), int(k_offset), _stream(q.device)))
    _count(1)
    return out, lse


def _segs(segs):
    arr = (_lib.Segment * max(1, len(segs)))()
    for i, (row0, rows, pos0) in enumerate(segs):
        arr[i] = _lib.Segment(int(row0), int(rows), int(pos0))
    return arr


def attention_segments(q, k, v, q_segs, kv_segs, causal, out, lse):
    """Every q segment (row0, rows, pos0) against the union of the kv segments
    in one launch; writes out/lse rows of the q segments only.  ``out`` is a
    bf16 block buffer, or a float32 accumulator that these rows are the first
    contribution to (written directly, replacing init + merge)."""
    _check_qkv(q, k, v)
    if not isinstance(out, torch.Tensor) or out.dtype not in (torch.bfloat16, torch.float32):
        raise DimensionError("out must be a bf16 or float32 tensor")
    _require_cuda("out", out, out.dtype)
    _require_cuda("lse", lse, torch.float32)
    if out.shape != q.shape or lse.shape != (q.shape[1], q.shape[0]):
        raise DimensionError("out/lse must match q's (T,H,D) / (H,T)")
    qs, ks = _segs(q_segs), _segs(kv_segs)
    dt = _lib.TR_DTYPE_F32 if out.dtype == torch.float32 else _lib.TR_DTYPE_BF16
    with _on(q):
        _lib.check(_lib.lib().tr_attention_segments(
            _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), q.shape[0], k.shape[0], q.shape[1],
            q.shape[2], qs, len(q_segs), ks, len(kv_segs), 1 if causal else 0, dt,
            _stream(q.device)))
    _count(1)
    return out, lse


def attention_segments_push(q, k, v, q_segs, kv_segs, causal, out, lse, row_shift,
                            done_count=None, done_flag=None, done_value=0, epoch=None):
    """``attention_segments`` whose epilogue writes straight into a message
    receive buffer -- typically the home rank's, mapped over CUDA IPC, so the
    OUT_LSE message of the next step (ref engine.py:346-353) travels over
    NVLink while the grid still computes.  ``out`` (n, H, D) bf16 and ``lse``
    (H, n) float32 hold q rows [row_shift, row_shift + n).  With
    ``done_flag`` (an int64 device tensor element, possibly a peer's) the
    kernel's last CTA raises it to ``done_value``; ``done_count`` is a zeroed
    int32 device counter owned by the caller's stream.  With ``epoch`` (a
    one-element int64 device tensor) ``done_value`` is an offset: the flag is
    raised to ``epoch + done_value`` as the epoch reads when the kernel ends
    (CUDA-graph replays; tr_attention_segments_push_rel)."""
    _check_qkv(q, k, v)
    _require_cuda("out", out, torch.bfloat16)
    _require_cuda("lse", lse, torch.float32)
    n = out.shape[0]
    if out.dim() != 3 or out.shape[1:] != q.shape[1:] or lse.shape != (q.shape[1], n):
        raise DimensionError("out/lse must be (n,H,D) / (H,n) with q's H and D")
    for r0, rows, _ in q_segs:
        if rows and (r0 < row_shift or r0 + rows - row_shift > n):
            raise DimensionError(f"q rows [{r0}, {r0 + rows}) do not fit the receive buffer "
                                 f"at shift {row_shift} (n={n})")
    if (done_flag is None) != (done_count is None):
        raise DimensionError("done_flag and done_count go together")
    if done_flag is not None:
        _require_cuda("done_flag", done_flag, torch.int64)
        _require_cuda("done_count", done_count, torch.int32)
    qs, ks = _segs(q_segs), _segs(kv_segs)
    with _on(q):
        if epoch is not None:
            if done_flag is None:
                raise DimensionError("epoch needs done_flag")
            _require_cuda("epoch", epoch, torch.int64)
            _lib.check(_lib.lib().tr_attention_segments_push_rel(
                _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), q.shape[0], k.shape[0],
                q.shape[1], q.shape[2], qs, len(q_segs), ks, len(kv_segs), 1 if causal else 0,
                row_shift, n, _ptr(done_count), _ptr(done_flag), _ptr(epoch), int(done_value),
                _stream(q.device)))
        else:
            _lib.check(_lib.lib().tr_attention_segments_push(
                _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), q.shape[0], k.shape[0],
                q.shape[1], q.shape[2], qs, len(q_segs), ks, len(kv_segs), 1 if causal else 0,
                row_shift, n, None if done_count is None else _ptr(done_count),
                None if done_flag is None else _ptr(done_flag), done_value, _stream(q.device)))
    _count(1)
    return out, lse


TR_LAUNCH_AFTER_PREV, TR_LAUNCH_RELEASE_NEXT = 1, 2


class overlap_launches:
    """Context manager (tr_set_launch_overlap) for the launches made inside it
    on this thread.  ``after_prev``: the D=64/128 attention launches and flag
    waits/sets are programmatic dependent launches of the previous kernel on
    their stream -- their CTAs take the SMs the previous grid's last wave
    frees instead of waiting for the whole grid; only for launches that read
    nothing the previous kernel writes (TokenRing steps whose messages were
    waited for by an earlier kernel).  ``release_next``: the attention
    launches let such a dependent start as soon as all their CTAs are
    resident (otherwise it starts when the grid ends)."""

    def __init__(self, after_prev=True, release_next=True):
        self.flags = ((TR_LAUNCH_AFTER_PREV if after_prev else 0)
                      | (TR_LAUNCH_RELEASE_NEXT if release_next else 0))

    def __enter__(self):
        self.prev = _lib.lib().tr_set_launch_overlap(self.flags)
        return self

    def __exit__(self, *exc):
        _lib.lib().tr_set_launch_overlap(self.prev)
        return False


def merge_state_(acc_out, acc_lse, blk_out, blk_lse, final_out=None):
    """In place: acc <- merge(acc, blk).  acc_out float32 (T,H,D); acc_lse /
    blk_lse may be column slices of wider (H, S) buffers (row stride S)."""
    _require_cuda("acc_out", acc_out, torch.float32)
    if not isinstance(blk_out, torch.Tensor) or not blk_out.is_cuda or not blk_out.is_contiguous():
        raise DimensionError("blk_out must be a contiguous CUDA tensor")
    if blk_out.dtype not in (torch.bfloat16, torch.float32):
        raise DimensionError("blk_out must be bf16 or float32")
    if acc_out.shape != blk_out.shape:
        raise DimensionError(
            f"cannot merge partials of shape {tuple(acc_out.shape)} and {tuple(blk_out.shape)}")
    t, h, d = acc_out.shape
    for n, l in (("acc_lse", acc_lse), ("blk_lse", blk_lse)):
        if l.dtype != torch.float32 or l.shape != (h, t) or l.stride(1) != 1:
            raise DimensionError(f"{n} must be float32 (H, T) with unit column stride")
    dt = _lib.TR_DTYPE_BF16 if blk_out.dtype == torch.bfloat16 else _lib.TR_DTYPE_F32
    fin = None
    if final_out is not None:
        _require_cuda("final_out", final_out, torch.bfloat16)
        fin = _ptr(final_out)
    with _on(acc_out):
        _lib.check(_lib.lib().tr_merge_state(
            _ptr(acc_out), _ptr(acc_lse), _ptr(blk_out), dt, _ptr(blk_lse), t, h, d,
            acc_lse.stride(0), blk_lse.stride(0), fin, _stream(acc_out.device)))
    _count(2)
    return acc_out, acc_lse


def merge_n_(acc_out, acc_lse, blocks, final_out=None):
    """In place: acc <- merge(acc, *blocks) in one pass per TR_MERGE_MAX
    blocks (tr_merge_n).  ``blocks``: [(blk_out, blk_lse)], blk_out bf16 or
    float32 (T,H,D) contiguous (all the same dtype), blk_lse float32 (H, T)
    with unit column stride (column slices of wider buffers are fine)."""
    _require_cuda("acc_out", acc_out, torch.float32)
    t, h, d = acc_out.shape
    if acc_lse.dtype != torch.float32 or acc_lse.shape != (h, t) or acc_lse.stride(1) != 1:
        raise DimensionError("acc_lse must be float32 (H, T) with unit column stride")
    dtypes = {bo.dtype for bo, _ in blocks}
    if len(dtypes) > 1 or not dtypes <= {torch.bfloat16, torch.float32}:
        raise DimensionError("blocks must all be bf16 or all float32")
    for bo, bl in blocks:
        if not bo.is_cuda or not bo.is_contiguous() or bo.shape != acc_out.shape:
            raise DimensionError(f"block of shape {tuple(bo.shape)} does not match the "
                                 f"accumulator {tuple(acc_out.shape)}")
        if bl.dtype != torch.float32 or bl.shape != (h, t) or bl.stride(1) != 1:
            raise DimensionError("block lse must be float32 (H, T) with unit column stride")
    if final_out is not None:
        _require_cuda("final_out", final_out, torch.bfloat16)
    dt = _lib.TR_DTYPE_F32 if dtypes == {torch.float32} else _lib.TR_DTYPE_BF16
    groups = [blocks[i:i + _lib.TR_MERGE_MAX] for i in range(0, len(blocks), _lib.TR_MERGE_MAX)]
    for gi, grp in enumerate(groups or [[]]):
        n = len(grp)
        outs = (ctypes.c_void_p * max(1, n))(*[bo.data_ptr() for bo, _ in grp])
        lses = (ctypes.c_void_p * max(1, n))(*[bl.data_ptr() for _, bl in grp])
        strides = (ctypes.c_int64 * max(1, n))(*[bl.stride(0) for _, bl in grp])
        fin = _ptr(final_out) if final_out is not None and gi == len(groups or [[]]) - 1 else None
        with _on(acc_out):
            _lib.check(_lib.lib().tr_merge_n(
                _ptr(acc_out), _ptr(acc_lse), acc_lse.stride(0), outs, dt, lses, strides, n, t, h,
                d, fin, _stream(acc_out.device)))
        _count(2)
    return acc_out, acc_lse


def merge_state(acc_out, acc_lse, blk_out, blk_lse):
    out = acc_out.to(torch.float32, copy=True).contiguous()
    lse = acc_lse.to(torch.float32, copy=True).contiguous()
    return merge_state_(out, lse, blk_out.contiguous(), blk_lse.to(torch.float32).contiguous())


def partial_init_(acc_out, acc_lse):
    _require_cuda("acc_out", acc_out, torch.float32)
    _require_cuda("acc_lse", acc_lse, torch.float32)
    t, h, d = acc_out.shape
    if tuple(acc_lse.shape) != (h, t):
        raise DimensionError(f"acc_lse must be {(h, t)}, got {tuple(acc_lse.shape)}")
    with _on(acc_out):
        _lib.check(_lib.lib().tr_partial_init(_ptr(acc_out), _ptr(acc_lse), t, h, d,
                                              _stream(acc_out.device)))
    _count(1)
    return acc_out, acc_lse


def splitmix_bf16_(dst, seed, first, low=-1.0, high=1.0):
    """Fill contiguous bf16 ``dst`` with SplitMix64 draws first.. of ``seed``."""
    _require_cuda("dst", dst, torch.bfloat16)
    with _on(dst):
        _lib.check(_lib.lib().tr_splitmix_bf16(
            ctypes.c_uint64(int(seed) % (1 << 64)), int(first), dst.numel(), float(low),
            float(high), _ptr(dst), _stream(dst.device)))
    _count(1)
    return dst


def flag_set_(flag, value, stream=None, epoch=None):
    """Raise a (possibly peer-mapped) int64 sequence flag after all prior work
    on ``stream`` (system-scope release store).  With ``epoch`` (one-element
    int64 device tensor) the value is ``epoch + value``, read on the device."""
    s = stream or torch.cuda.current_stream(flag.device)
    with torch.cuda.device(s.device):
        if epoch is None:
            _lib.check(_lib.lib().tr_flag_set(_ptr(flag), int(value),
                                              ctypes.c_void_p(s.cuda_stream)))
        else:
            _lib.check(_lib.lib().tr_flag_set_rel(_ptr(flag), _ptr(epoch), int(value),
                                                  ctypes.c_void_p(s.cuda_stream)))
    _count(1)


def flag_wait_(flag, value, stream=None, epoch=None):
    """Make ``stream`` wait until ``flag >= value`` (one-thread acquire spin);
    with ``epoch``, until ``flag >= epoch + value``."""
    s = stream or torch.cuda.current_stream(flag.device)
    with torch.cuda.device(s.device):
        if epoch is None:
            _lib.check(_lib.lib().tr_flag_wait(_ptr(flag), int(value),
                                               ctypes.c_void_p(s.cuda_stream)))
        else:
            _lib.check(_lib.lib().tr_flag_wait_rel(_ptr(flag), _ptr(epoch), int(value),
                                                   ctypes.c_void_p(s.cuda_stream)))
    _count(1)


def epoch_add_(epoch, delta, stream=None):
    """epoch += delta on the device, in ``stream`` order (the last operation of
    a captured forward: the next replay's flag values move on by delta)."""
    s = stream or torch.cuda.current_stream(epoch.device)
    with torch.cuda.device(s.device):
        _lib.check(_lib.lib().tr_epoch_add(_ptr(epoch), int(delta),
                                           ctypes.c_void_p(s.cuda_stream)))
    _count(1)


def copy_(dst, src, stream=None):
    """Copy-engine transfer (cudaMemcpyAsync, UVA) between contiguous tensors,
    local or peer-mapped; no SMs are used."""
    if dst.numel() * dst.element_size() != src.numel() * src.element_size():
        raise DimensionError("copy_ size mismatch")
    if not (dst.is_contiguous() and src.is_contiguous()):
        raise DimensionError("copy_ needs contiguous tensors")
    s = stream or torch.cuda.current_stream(src.device)
    with torch.cuda.device(s.device):
        _lib.check(_lib.lib().tr_copy_async(_ptr(dst), _ptr(src), dst.numel() * dst.element_size(),
                                            ctypes.c_void_p(s.cuda_stream)))


def enable_peer_access(peer_device):
    """Let kernels on the current device dereference ``peer_device`` memory
    (IPC-mapped flags / receive slots of the ipc and fused transports)."""
    _lib.check(_lib.lib().tr_enable_peer_access(int(peer_device)))


def poll_error():
    """Raise ScheduleError if a flag wait of this process has timed out (a
    message that never arrived; the library records it instead of trapping).
    Reads pinned host memory only -- no device synchronisation."""
    _lib.check(_lib.lib().tr_poll_error())


def clear_error():
    _lib.lib().tr_clear_error()


def set_flag_timeout_ms(ms):
    """Timeout of later flag waits (default 30 s); for tests of the failure path."""
    _lib.lib().tr_set_flag_timeout_ms(int(ms))
