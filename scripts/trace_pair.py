"""TR_TRACE timeline of the CTA-pair kernel (build: -D TR_KERNEL_PAIR -D TR_TRACE):
leader MMA warp vs the softmax warps of both CTAs (globaltimer for cross-SM)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _ablib import maybe_use_env_library  # noqa: E402
maybe_use_env_library()
from paper_2412_20501_b200 import _lib, kernels as K  # noqa: E402

tq, tk, h, d = 8192, 16384, 32, 128
q = torch.randn(tq, h, d, device="cuda").to(torch.bfloat16) * 0.5
k = torch.randn(tk, h, d, device="cuda").to(torch.bfloat16) * 0.5
v = torch.randn(tk, h, d, device="cuda").to(torch.bfloat16)
for _ in range(3):
    K.attention_block(q, k, v, 0)
torch.cuda.synchronize()
buf = np.zeros(2 * 20 * 64 * 8, dtype=np.uint64)
L = _lib.lib()
L.tr_debug_trace_variants.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.tr_debug_trace_variants(buf.ctypes.data, buf.nbytes) == 0
t = buf.reshape(2, 20, 64, 8).astype(np.int64)
J = slice(8, 60)
MW = int(os.environ.get("MMA_WARP", 1))
mma = t[0, MW]
print("MMA (leader, clock64): iter start -> V landed", np.median(mma[J, 4] - mma[J, 0]),
      " V -> P_A seen", np.median(mma[J, 1] - mma[J, 4]), " P_A -> P_B", np.median(mma[J, 2] - mma[J, 1]),
      " P_B -> end", np.median(mma[J, 3] - mma[J, 2]), " period", np.median(np.diff(mma[8:60, 0])))
for cta in (0, 1):
    for w in (4, 8):
        s = t[cta, w]
        print(f"cta {cta} warp {w}: period {np.median(np.diff(s[8:60, 1])):.0f} S ready->max "
              f"{np.median(s[J, 2] - s[J, 1]):.0f} max->P done {np.median(s[J, 3] - s[J, 2]):.0f} "
              f"P done->next S ready {np.median(s[9:61, 1] - s[J, 3]):.0f}")
# globaltimer (ns): softmax P published (slot 5) in both CTAs vs MMA P_A seen (slot 5)
seen = t[0, MW][J, 5]
for cta in (0, 1):
    for w in (4, 5, 6, 7, 8, 9, 10, 11):
        pub = t[cta, w][J, 5]
        print(f"  cta {cta} warp {w:2d}: MMA sees P_A  {np.median(seen - pub):7.0f} ns after this warp published")
print("leader CTA, per warp (clock64, relative to warp 4): S ready, max done, P done")
base = t[0, 4][J]
for w in range(4, 12):
    s = t[0, w][J]
    print(f"  warp {w:2d}: {np.median(s[:, 1] - base[:, 1]):6.0f} {np.median(s[:, 2] - base[:, 2]):6.0f} "
          f"{np.median(s[:, 3] - base[:, 3]):6.0f}")
