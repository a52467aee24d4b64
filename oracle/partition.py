"""Token partitions (oracle; test infrastructure only).

Restates ``pkg/src/ringsim/partition.py``:
* contiguous slabs, P | S                    (ref :57-66)
* zigzag: rank r owns chunks r, 2P-1-r       (ref :69-84)
* exact causal pair counts per rank          (ref :87-100)
* gather / global reorder                    (ref :103-135)
Ranges are returned as tuples of (start, stop) per rank, ascending.
"""

import numpy as np


class OracleConfigError(ValueError):
    pass


def contiguous(seq_len, ranks):
    if ranks < 1 or seq_len < ranks or seq_len % ranks:
        raise OracleConfigError("ranks must divide seq_len")
    n = seq_len // ranks
    return tuple(((r * n, (r + 1) * n),) for r in range(ranks))


def zigzag(seq_len, ranks):
    if ranks < 1 or seq_len % (2 * ranks):
        raise OracleConfigError("2P must divide seq_len")
    c = seq_len // (2 * ranks)
    return tuple(((r * c, (r + 1) * c), ((2 * ranks - 1 - r) * c, (2 * ranks - r) * c))
                 for r in range(ranks))


def causal_pairs(ranges_per_rank):
    # sum over q in [a, b) of (q + 1)
    return tuple(sum((b * (b + 1) - a * (a + 1)) // 2 for a, b in rr)
                 for rr in ranges_per_rank)


def gather(arr, ranges):
    return np.concatenate([arr[a:b] for a, b in ranges], axis=0)


def reorder(outs, lses, ranges_per_rank, seq_len):
    """Per-rank (out (T_r,H,D), lse (H,T_r)) -> global (S,H,D), (H,S)."""
    h, d = outs[0].shape[1], outs[0].shape[2]
    out = np.empty((seq_len, h, d))
    lse = np.empty((h, seq_len))
    for r, rr in enumerate(ranges_per_rank):
        cur = 0
        for a, b in rr:
            out[a:b] = outs[r][cur:cur + b - a]
            lse[:, a:b] = lses[r][:, cur:cur + b - a]
            cur += b - a
    return out, lse
