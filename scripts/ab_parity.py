"""Parity gate for an A/B library build (never the product path): the block
attention of the library TOKENRING_LIB points at, against a float32 torch
reference of the same op, on a causal and a ragged non-causal shape.

    TOKENRING_LIB=paper_2412_20501_b200/_variants/lib_x.so python scripts/ab_parity.py
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


def ref(q, k, v, causal):
    qf, kf, vf = (x.float().permute(1, 0, 2) for x in (q, k, v))
    s = qf @ kf.transpose(1, 2) / math.sqrt(q.shape[-1])
    if causal:
        tq, tk = q.shape[0], k.shape[0]
        m = torch.arange(tk, device=q.device)[None, :] > torch.arange(tq, device=q.device)[:, None]
        s = s.masked_fill(m, float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ vf
    return o.permute(1, 0, 2), lse


def main():
    torch.manual_seed(0)
    worst = 0.0
    for tq, tk, h, causal, scale in ((4096, 4096, 4, True, 0.5), (1000, 3000, 4, False, 0.5),
                                     (2048, 2048, 2, True, 3.0)):
        q = (torch.randn(tq, h, 128, device="cuda") * scale).to(torch.bfloat16)
        k = (torch.randn(tk, h, 128, device="cuda") * scale).to(torch.bfloat16)
        v = torch.randn(tk, h, 128, device="cuda").to(torch.bfloat16)
        out, lse = K.attention_block(q, k, v, 2 if causal else 0, 0, 0)
        ro, rl = ref(q, k, v, causal)
        eo = (out.float() - ro).abs().max().item()
        el = (lse - rl).abs().max().item()
        worst = max(worst, eo / 2e-2, el / 1e-3)
        print(f"{tq}x{tk} H={h} causal={causal} scale={scale}: out {eo:.3e} lse {el:.3e}")
    print(f"{lib or 'product'}: {'PASS' if worst <= 1 else 'FAIL'}")
    sys.exit(0 if worst <= 1 else 1)


if __name__ == "__main__":
    main()
