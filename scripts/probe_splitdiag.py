import os, sys, torch
sys.path.insert(0, "scripts"); sys.path.insert(0, ".")
from _ablib import maybe_use_env_library
lib = maybe_use_env_library()
from paper_2412_20501_b200 import kernels as K
from probe_step0 import timed
H, D = 32, 128
for tq, tk in ((2048, 4096), (4096, 2048)):
    q = (torch.randn(tq, H, D, device="cuda") * 0.5).to(torch.bfloat16)
    k = (torch.randn(tk, H, D, device="cuda") * 0.5).to(torch.bfloat16)
    v = torch.randn(tk, H, D, device="cuda").to(torch.bfloat16)
    o = torch.empty(tq, H, D, device="cuda", dtype=torch.bfloat16); l = torch.empty(H, tq, device="cuda")
    ms = timed(lambda: K.attention_block(q, k, v, 0, out=o, lse=l))
    print(f"{lib or 'product'} {tq}x{tk}: {ms*1e3:.1f} us")
