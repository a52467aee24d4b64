"""Device-time probe of the lse-merge kernel at the TokenRing return size
(2 sub-chunks of c=8192 rows, H=32, D=128: a config-3 OUT_LSE payload).
Algorithmic bytes per merge = T*H*(D*(4+2+4) + 3*4): read the float32
accumulator, read the bf16 block, write the accumulator, plus three lse
streams."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20501_b200 import kernels as K  # noqa: E402


def main(T=16384, H=32, D=128, iters=20):
    acc = torch.randn(T, H, D, device="cuda")
    al = torch.randn(H, T, device="cuda")
    blk = torch.randn(T, H, D, device="cuda").to(torch.bfloat16)
    bl = torch.randn(H, T, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        K.merge_state_(acc, al, blk, bl)
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(iters):
        flush.zero_()            # > L2: every merge starts cold
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        K.merge_state_(acc, al, blk, bl)
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    ms = tot / iters
    nbytes = T * H * (D * (4 + 2 + 4) + 12)
    print(f"merge T={T} H={H} D={D}: {ms:.4f} ms, {nbytes / ms / 1e6:.1f} GB/s algorithmic")


def main_n(c=8192, H=32, D=128, n=7, iters=20):
    """Config-3 home chunk (c rows) receiving n=P-1 returned partials:
    n pairwise merges vs one tr_merge_n (bytes: c*H*(D*(4 + 2n + 4) + 4(n+2)))."""
    acc = torch.randn(c, H, D, device="cuda")
    al = torch.randn(H, c, device="cuda")
    blks = [(torch.randn(c, H, D, device="cuda").to(torch.bfloat16), torch.randn(H, c, device="cuda"))
            for _ in range(n)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def pairwise():
        for bo, bl in blks:
            K.merge_state_(acc, al, bo, bl)

    def nway():
        K.merge_n_(acc, al, blks)

    for name, fn in (("pairwise", pairwise), ("n-way", nway)):
        for _ in range(3):
            fn()
        tot = 0.0
        for _ in range(iters):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            tot += s.elapsed_time(e)
        ms = tot / iters
        nbytes = c * H * (D * (4 + 2 * n + 4) + 4 * (n + 2))
        print(f"{name:8s} c={c} H={H} D={D} n={n}: {ms:.4f} ms"
              + (f", {nbytes / ms / 1e6:.1f} GB/s algorithmic" if name == "n-way" else ""))


if __name__ == "__main__":
    main()
    main_n()
