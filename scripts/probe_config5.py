"""Config 5 (Llama-70B attention shape: S=1,048,576, H=64, D=128, causal) on
one B200: the whole sequence as ONE causal launch (what one GPU would do
without sequence parallelism), timed with CUDA events; algorithmic flops
4*H*D*S(S+1)/2 (ref engine.py:170-173).

    python scripts/probe_config5.py [--iters 2]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20501_b200 import kernels as K, rng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--seq", type=int, default=1 << 20)
    ap.add_argument("--heads", type=int, default=64)
    a = ap.parse_args()
    S, H, D = a.seq, a.heads, 128
    q, k, v = rng.attention_inputs(0, S, H, D, device="cuda")
    out = torch.empty((S, H, D), dtype=torch.float32, device="cuda")
    lse = torch.empty((H, S), dtype=torch.float32, device="cuda")
    segs = [(0, S, 0)]
    K.attention_segments(q, k, v, segs, segs, True, out, lse)     # warm-up
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.iters):
        K.attention_segments(q, k, v, segs, segs, True, out, lse)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.iters
    flops = 4 * H * D * (S * (S + 1) // 2)
    print(json.dumps({"workload": f"causal S={S} H={H} D={D} one launch, f32 out", "ms": ms,
                      "tflops": flops / ms / 1e9, "tokens_per_s": S / ms * 1e3}))


if __name__ == "__main__":
    main()
