"""TR_TRACE timeline of the split-row pair kernel (TR_PAIR2_SPLIT build):
CTA 0, per half the slowest of its 8 softmax warps (two per lane quarter,
one per 64-key half): S ready -> max exchanged -> P published, the MMA's
view, and the period (cycles, medians over steady-state tiles)."""
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
L.tr_debug_trace_pair2.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.tr_debug_trace_pair2(buf.ctypes.data, buf.nbytes) == 0
t = buf.reshape(2, 20, 64, 8).astype(np.int64)[0]
J = np.arange(8, 56)
mma = t[1]
med = lambda x: float(np.median(x))  # noqa: E731
print(f"split kernel, shape {tq}x{tk} H={h}; CTA 0; medians over tiles 8..55 (cycles)")
print(f"MMA period: {med(np.diff(mma[8:57, 0]))}")
for half, groups, seen in ((0, ((4, 5, 6, 7), (12, 13, 14, 15)), (4, 5)), (1, ((8, 9, 10, 11), (16, 17, 18, 19)), (1, 2))):
    for kc, ws in enumerate(groups):
        sw = t[list(ws)]
        s_ready = sw[:, J, 1].min(0)
        mx = sw[:, J, 2].max(0)
        pub = sw[:, J, 3].max(0)
        nxt = sw[:, J + 1, 1].min(0)
        ms = mma[J, seen[kc]]
        print(f"half {half} keys {64 * kc}-{64 * kc + 63}: S ready -> max exch {med(mx - s_ready):.0f} "
              f"-> P pub {med(pub - mx):.0f} | pub -> MMA sees {med(ms - pub):.0f} | MMA sees -> next S "
              f"ready {med(nxt - ms):.0f} | period {med(np.diff(sw[0, 8:57, 1])):.0f}")
