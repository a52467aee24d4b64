"""Fixed cost of one CTA-pair work item: launches of exactly one wave (74
pair tiles of 512 rows = 148 CTAs) over n kv tiles of 128 keys, non-causal;
time(n) = a + n * t, so the intercept a is launch + per-item prologue and
epilogue and t the steady-state kv-tile period.  Diagnostic only.

    python scripts/probe_overhead.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _ablib import maybe_use_env_library  # noqa: E402
maybe_use_env_library()
from paper_2412_20501_b200 import kernels as K  # noqa: E402


def timed(fn, n=30, batch=20):
    """Median per-launch device time of `batch` back-to-back launches (the
    host enqueues ahead of the GPU, as in a TokenRing step loop, after a
    sleep kernel gives it a head start)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        a.record()
        for _ in range(batch):
            fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / batch)
    ts.sort()
    return ts[len(ts) // 2] * 1e3


def main():
    H, D = 2, 128
    tq = 37 * 512                      # 37 pair tiles per head x 2 heads = 74 pairs
    q = (torch.randn(tq, H, D, device="cuda") * 0.5).to(torch.bfloat16)
    kmax = 128 * 256
    k = (torch.randn(kmax, H, D, device="cuda") * 0.5).to(torch.bfloat16)
    v = torch.randn(kmax, H, D, device="cuda").to(torch.bfloat16)
    out = torch.empty(tq, H, D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, tq, device="cuda")
    pts = []
    for n in (1, 2, 4, 8, 16, 32, 64, 128, 256):
        kk, vv = k[:128 * n], v[:128 * n]
        us = timed(lambda: K.attention_block(q, kk, vv, 0, out=out, lse=lse))
        pts.append((n, us))
        print(f"n={n:4d} kv tiles: {us:9.1f} us")
    # least squares over n >= 8
    xs = [n for n, _ in pts if n >= 8]
    ys = [u for n, u in pts if n >= 8]
    mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
    t = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
    a = my - t * mx
    print(f"fit n>=8: time = {a:.1f} us + n * {t:.3f} us  (fixed cost = {a / t:.1f} kv-tile periods)")
    torch.cuda.synchronize()
    # empty launch cost for reference
    e = torch.empty(0, device="cuda")
    us = timed(lambda: e.add_(1))
    print(f"torch empty-kernel launch: {us:.1f} us")


if __name__ == "__main__":
    main()
