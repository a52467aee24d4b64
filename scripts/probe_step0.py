"""Why is a zigzag step 0 slow at small S?  Times single launches (median of
20, CUDA events) of: the rank-0 step-0 geometry of zigzag TokenRing (two q
segments x two kv segments, causal), one causal block of the same rows, and a
full (non-causal) block with the same useful pairs.  Diagnostic only.

    python scripts/probe_step0.py [S] [P]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _ablib import maybe_use_env_library  # noqa: E402
maybe_use_env_library()
from paper_2412_20501_b200 import kernels as K  # noqa: E402


def timed(fn, n=15, batch=20):
    """Median per-launch device time of `batch` back-to-back launches (the
    host enqueues ahead of the GPU after a sleep kernel's head start, as in a
    step loop; a single launch on an idle GPU would time the host's launch
    path too)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(5_000_000)
        a.record()
        for _ in range(batch):
            fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / batch)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    H, D = 32, 128
    c = S // (2 * P)                      # zigzag chunk
    n = 2 * c                             # rows per rank
    q = (torch.randn(n, H, D, device="cuda") * 0.5).to(torch.bfloat16)
    k = (torch.randn(n, H, D, device="cuda") * 0.5).to(torch.bfloat16)
    v = torch.randn(n, H, D, device="cuda").to(torch.bfloat16)
    out = torch.empty(n, H, D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, n, device="cuda")
    acc = torch.empty(n, H, D, device="cuda", dtype=torch.float32)
    for r in (0, P // 2, P - 1):
        segs = [(0, c, r * c), (c, c, (2 * P - 1 - r) * c)]
        useful = c * (c + 1) // 2 * 2 + c * c      # two causal diagonals + one full block
        ms = timed(lambda: K.attention_segments(q, k, v, segs, segs, True, out, lse))
        print(f"step0 rank {r}: 2 q segs x 2 kv segs of {c} rows, causal: {ms * 1e3:8.1f} us  "
              f"{4 * H * D * useful / ms / 1e9:7.1f} TF")
        ms = timed(lambda: K.attention_segments(q, k, v, segs, segs, True, acc, lse))
        print(f"   same, float32 rows into the accumulator:       {ms * 1e3:8.1f} us  "
              f"{4 * H * D * useful / ms / 1e9:7.1f} TF")
    ms = timed(lambda: K.attention_block(q, k, v, 2, 0, 0, out=out, lse=lse))
    print(f"one causal block of {n} rows:                  {ms * 1e3:8.1f} us  "
          f"{4 * H * D * (n * (n + 1) // 2) / ms / 1e9:7.1f} TF")
    qh = q[:c]
    o2 = torch.empty(c, H, D, device="cuda", dtype=torch.bfloat16)
    l2 = torch.empty(H, c, device="cuda")
    ms = timed(lambda: K.attention_block(qh, k, v, 0, out=o2, lse=l2))
    print(f"full block {c} x {n}:                          {ms * 1e3:8.1f} us  "
          f"{4 * H * D * c * n / ms / 1e9:7.1f} TF")
    ms = timed(lambda: K.attention_block(q, k[:c], v[:c], 0, out=out, lse=lse))
    print(f"full block {n} x {c}:                          {ms * 1e3:8.1f} us  "
          f"{4 * H * D * c * n / ms / 1e9:7.1f} TF")


if __name__ == "__main__":
    main()
