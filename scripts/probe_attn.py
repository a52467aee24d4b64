"""Quick device-time probe of the attention kernel (not the bench contract).

    python scripts/probe_attn.py [--iters 10]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _ablib import maybe_use_env_library  # noqa: E402
maybe_use_env_library()
from paper_2412_20501_b200 import kernels as K  # noqa: E402


def bench(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--case", type=int, nargs="*", default=[], help="run only these case indices")
    a = ap.parse_args()
    cases = [
        ("causal S=32768 H=32 D=128", 32768, 32768, 32, 128, 2),
        ("full 8192x16384 H=32 D=128", 8192, 16384, 32, 128, 0),
        ("full 16384x8192 H=32 D=128", 16384, 8192, 32, 128, 0),
        ("causal S=131072 H=32 D=128", 131072, 131072, 32, 128, 2),
        ("full 4096x4096 H=8 D=64", 4096, 4096, 8, 64, 0),
        # per-CTA fixed cost: same flops, 256 / 128 / 64 / 32 kv tiles per CTA
        ("full 4096x32768 H=32 D=128", 4096, 32768, 32, 128, 0),
        ("full 8192x16384 H=32 D=128", 8192, 16384, 32, 128, 0),
        ("full 16384x8192 H=32 D=128", 16384, 8192, 32, 128, 0),
        ("full 32768x4096 H=32 D=128", 32768, 4096, 32, 128, 0),
    ]
    if a.case:
        cases = [cases[i] for i in a.case]
    for name, tq, tk, h, d, mask in cases:
        q = torch.randn(tq, h, d, device="cuda").to(torch.bfloat16) * 0.5
        k = torch.randn(tk, h, d, device="cuda").to(torch.bfloat16) * 0.5
        v = torch.randn(tk, h, d, device="cuda").to(torch.bfloat16)
        out = torch.empty_like(q)
        lse = torch.empty(h, tq, device="cuda")
        ms = bench(lambda: K.attention_block(q, k, v, mask, 0, 0, out=out, lse=lse),
                   a.iters if tq < 100000 else 2)
        pairs = tq * (tq + 1) // 2 if mask == 2 else tq * tk
        fl = 4 * h * d * pairs
        print(f"{name:32s} {ms:9.3f} ms  {fl / ms / 1e9:8.1f} TFLOP/s")


if __name__ == "__main__":
    main()
