"""Synthetic inputs on the device, bit-exact with ``ringsim.rng``
(``pkg/src/ringsim/rng.py:25-53``) after the canonical fp64 -> fp32 -> bf16
rounding.  q, k, v are consecutive slices of one SplitMix64 stream of
3*S*H*D draws; a rank can materialise just its own rows (zigzag shards of a
1M-token sequence never exist in full anywhere)."""

import torch

from . import kernels


def attention_rows(seed, seq_len, heads, head_dim, which, ranges, low=-1.0, high=1.0,
                   device=None):
    """Rows of tensor ``which`` (0=q, 1=k, 2=v) for the given global token
    ranges, concatenated in order, as a bf16 (rows, H, D) CUDA tensor."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    per_row = heads * head_dim
    n = seq_len * per_row
    rows = sum(b - a for a, b in ranges)
    out = torch.empty((rows, heads, head_dim), dtype=torch.bfloat16, device=device)
    cur = 0
    for a, b in ranges:
        kernels.splitmix_bf16_(out[cur:cur + b - a], seed, which * n + a * per_row, low, high)
        cur += b - a
    return out


def attention_inputs(seed, seq_len, heads, head_dim, low=-1.0, high=1.0, device=None):
    """Full (q, k, v), each (S, H, D) bf16 on the device."""
    full = ((0, seq_len),)
    return tuple(attention_rows(seed, seq_len, heads, head_dim, w, full, low, high, device)
                 for w in range(3))


def local_inputs(seed, part, rank, heads, head_dim, low=-1.0, high=1.0, device=None):
    """This rank's shard (its partition ranges, start order) of q, k, v."""
    rng = part.ranges(rank)
    return tuple(attention_rows(seed, part.seq_len, heads, head_dim, w, rng, low, high, device)
                 for w in range(3))
