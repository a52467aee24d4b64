"""Why is a zigzag TokenRing step 0 slower than the other steps?  Times the
step-0 launch of one rank at 128K / P=8 (c=8192, H=32, D=128: q chunks
{r, 2P-1-r} x kv chunks {r, 2P-1-r}, causal by position) and its pieces."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20501_b200 import kernels as K  # noqa: E402


def bench(fn, iters=10):
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


P, c, H, D, r = 8, 8192, 32, 128, 3
lo, hi = r * c, (2 * P - 1 - r) * c
q = torch.randn(2 * c, H, D, device="cuda").to(torch.bfloat16) * 0.5
k = torch.randn(2 * c, H, D, device="cuda").to(torch.bfloat16) * 0.5
v = torch.randn(2 * c, H, D, device="cuda").to(torch.bfloat16)
o16 = torch.empty(2 * c, H, D, device="cuda", dtype=torch.bfloat16)
o32 = torch.empty(2 * c, H, D, device="cuda", dtype=torch.float32)
lse = torch.empty(H, 2 * c, device="cuda")
segs = [(0, c, lo), (c, c, hi)]
cases = {
    "step0 f32 out (as run)": lambda: K.attention_segments(q, k, v, segs, segs, True, o32, lse),
    "step0 bf16 out": lambda: K.attention_segments(q, k, v, segs, segs, True, o16, lse),
    "lo x lo (diagonal)": lambda: K.attention_segments(q, k, v, segs[:1], segs[:1], True, o16, lse),
    "hi x {lo,hi}": lambda: K.attention_segments(q, k, v, segs[1:], segs, True, o16, lse),
    "hi x hi (diagonal)": lambda: K.attention_segments(q, k, v, segs[1:], segs[1:], True, o16, lse),
    "hi x lo (full)": lambda: K.attention_segments(q, k, v, segs[1:], segs[:1], True, o16, lse),
    "step>=1 shape: hi x {lo,hi} full": lambda: K.attention_segments(
        q, k, v, [(c, c, 2 * P * c)], segs, True, o16, lse),
}
flops = {"lo x lo (diagonal)": c * (c + 1) // 2, "hi x hi (diagonal)": c * (c + 1) // 2,
         "hi x lo (full)": c * c, "hi x {lo,hi}": c * c + c * (c + 1) // 2,
         "step>=1 shape: hi x {lo,hi} full": 2 * c * c}
flops["step0 f32 out (as run)"] = flops["step0 bf16 out"] = 2 * c * c + c
for name, fn in cases.items():
    ms = bench(fn)
    print(f"{name:36s} {ms:7.3f} ms  {4 * H * D * flops[name] / ms / 1e9:7.1f} TFLOP/s")
