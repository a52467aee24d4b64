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


if __name__ == "__main__":
    main()
