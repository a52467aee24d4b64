"""Dump the TR_TRACE timeline of CTA 0 (debug build lib_trace.so)."""
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
buf = np.zeros(12 * 64 * 8, dtype=np.uint64)
L = _lib.lib()
L.tr_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.tr_debug_trace(buf.ctypes.data, buf.nbytes) == 0
t = buf.reshape(12, 64, 8).astype(np.int64)
t0 = t[4, 4, 0]
J0, J1 = int(os.environ.get("J0", 4)), int(os.environ.get("J1", 12))
print("j | MMA0 slots 0-3 | MMA1 slots 0-3 | SM0: wait, S ready, max, P done | SM1: same")
for j in range(J0, J1):
    print(j, "|", *(int(x - t0) for x in t[1, j, 0:4]), "|", *(int(x - t0) for x in t[3, j, 0:4]),
          "|", *(int(x - t0) for x in t[4, j, :4]), "|", *(int(x - t0) for x in t[8, j, :4]))
for w in (4, 8):
    s = t[w]
    print(f"softmax warp {w}: period {np.median(np.diff(s[8:60, 1])):.0f}  S ready->max "
          f"{np.median(s[8:60, 2] - s[8:60, 1]):.0f}  max->P done {np.median(s[8:60, 3] - s[8:60, 2]):.0f}"
          f"  P done->next S ready {np.median(s[9:61, 1] - s[8:60, 3]):.0f}")
print("softmax phases (median cycles): S ready->max, max->half0 computed, ->half0 published, ->half1 computed, ->half1 published")
for w in (4, 5, 6, 7, 8):
    s = t[w][8:60]
    print(w, [int(np.median(s[:, b] - s[:, a])) for a, b in ((1, 2), (2, 4), (4, 5), (5, 6), (6, 7))])
