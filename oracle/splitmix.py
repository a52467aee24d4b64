"""SplitMix64 input stream (oracle; test infrastructure only).

Restates ``ringsim.rng`` (``pkg/src/ringsim/rng.py:25-53``): draw ``i`` of seed
``s`` is a pure hash of ``s + (i+1) * golden``; a double in [0,1) takes the top
53 bits; q, k, v are consecutive slices of one stream of 3*S*H*D draws.
"""

import numpy as np

_GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


def hash_draws(seed: int, start: int, count: int) -> np.ndarray:
    """Raw 64-bit draws ``start .. start+count-1`` (0-based) of ``seed``.

    ref rng.py:25-31 (there ``start`` is always 0)."""
    i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed % (1 << 64)) + i * np.uint64(_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


def unit_doubles(seed: int, start: int, count: int, low=0.0, high=1.0) -> np.ndarray:
    """ref rng.py:34-38: low + (high-low) * (z >> 11) * 2^-53."""
    u = (hash_draws(seed, start, count) >> np.uint64(11)).astype(np.float64)
    u *= 2.0 ** -53
    return low + (high - low) * u


def attention_inputs(seed, seq_len, heads, head_dim, low=-1.0, high=1.0):
    """ref rng.py:41-53: q, k, v of shape (S, H, D) from one stream."""
    n = seq_len * heads * head_dim
    shape = (seq_len, heads, head_dim)
    return tuple(unit_doubles(seed, j * n, n, low, high).reshape(shape)
                 for j in range(3))


def attention_rows(seed, seq_len, heads, head_dim, which, row0, rows,
                   low=-1.0, high=1.0):
    """Rows ``row0 .. row0+rows-1`` of tensor ``which`` (0=q, 1=k, 2=v)
    without materialising the whole stream (used for sampled parity at
    sizes where the full fp64 tensors would not fit in host memory)."""
    n = seq_len * heads * head_dim
    per_row = heads * head_dim
    flat = unit_doubles(seed, which * n + row0 * per_row, rows * per_row, low, high)
    return flat.reshape(rows, heads, head_dim)


def to_bf16_f64(x: np.ndarray) -> np.ndarray:
    """Round float64 -> bfloat16 (round-to-nearest-even via fp32) -> float64.

    The single canonical rounding path used on both sides of a parity check
    (fp64 -> fp32 -> bf16, RNE at each step)."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    b = ((b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
    return b.astype(np.uint32).view(np.float32).astype(np.float64)
