"""D=64 (the single-CTA tcgen05 kernel) throughput and parity on the library
TOKENRING_LIB points at (default: the product): back-to-back launches of a
full 8K x 16K and a causal 32K block, H=32, plus a float32 torch reference
check on a small causal shape.  Diagnostic only.

    python scripts/probe_d64.py
"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _ablib import maybe_use_env_library  # noqa: E402
lib = maybe_use_env_library()
from paper_2412_20501_b200 import kernels as K  # noqa: E402


def timed(fn, n=10, batch=10):
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
    H, D = 32, 64
    torch.manual_seed(0)
    for tq, tk, causal in ((8192, 16384, False), (32768, 32768, True)):
        q = (torch.randn(tq, H, D, device="cuda") * 0.5).to(torch.bfloat16)
        k = (torch.randn(tk, H, D, device="cuda") * 0.5).to(torch.bfloat16)
        v = torch.randn(tk, H, D, device="cuda").to(torch.bfloat16)
        out = torch.empty(tq, H, D, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(H, tq, device="cuda")
        ms = timed(lambda: K.attention_block(q, k, v, 2 if causal else 0, 0, 0, out=out, lse=lse))
        fl = 4 * H * D * (tq * (tq + 1) // 2 if causal else tq * tk)
        print(f"D=64 {'causal' if causal else 'full'} {tq}x{tk}: {ms * 1e3:8.1f} us  {fl / ms / 1e9:7.1f} TF")
    q = (torch.randn(2048, 4, D, device="cuda") * 0.5).to(torch.bfloat16)
    k = (torch.randn(2048, 4, D, device="cuda") * 0.5).to(torch.bfloat16)
    v = torch.randn(2048, 4, D, device="cuda").to(torch.bfloat16)
    o, l = K.attention_block(q, k, v, 2, 0, 0)
    qf, kf, vf = (x.float().permute(1, 0, 2) for x in (q, k, v))
    s = qf @ kf.transpose(1, 2) / math.sqrt(D)
    s = s.masked_fill(torch.ones(2048, 2048, device="cuda", dtype=torch.bool).triu(1), float("-inf"))
    ro = (torch.softmax(s, -1) @ vf).permute(1, 0, 2)
    rl = torch.logsumexp(s, -1)
    eo, el = (o.float() - ro).abs().max().item(), (l - rl).abs().max().item()
    print(f"{lib or 'product'} parity D=64 causal 2048: out {eo:.2e} lse {el:.2e} "
          f"{'PASS' if eo <= 2e-2 and el <= 1e-3 else 'FAIL'}")


if __name__ == "__main__":
    main()
