"""Kernel-vs-kernel check (diagnostic): run a few D=128 shapes through the
current library and save out/lse, so two runs with different kernel choices
(TR_ATTN_PAIR2=0/1, or TOKENRING_LIB=<variant build>) can be compared bitwise.

    TR_ATTN_PAIR2=0 python scripts/mc_check.py /tmp/a.pt
    TR_ATTN_PAIR2=1 python scripts/mc_check.py /tmp/b.pt
"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _ablib import maybe_use_env_library  # noqa: E402
maybe_use_env_library()
from paper_2412_20501_b200 import kernels as K
torch.manual_seed(0)
res = {}
for name, tq, tk, h, mask in [("full", 8192, 16384, 4, 0), ("causal", 4096, 4096, 4, 2), ("causal_odd", 3000, 3000, 2, 2)]:
    q = (torch.rand(tq, h, 128, device="cuda") * 2 - 1).bfloat16()
    k = (torch.rand(tk, h, 128, device="cuda") * 2 - 1).bfloat16()
    v = (torch.rand(tk, h, 128, device="cuda") * 2 - 1).bfloat16()
    try:
        o, l = K.attention_block(q, k, v, mask, 0, 0)
        torch.cuda.synchronize()
        res[name] = (o.float().cpu(), l.float().cpu())
    except Exception as e:
        res[name] = str(e)[:100]
torch.save(res, sys.argv[1])
