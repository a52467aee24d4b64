"""TR_TRACE timeline of CTA 0 for the P-in-smem kernel (debug build):
    python -m paper_2412_20501_b200.build -D TR_TRACE -D TR_PSMEM_DEFAULT=1 --out /tmp/ps_trace.so
    TOKENRING_LIB=/tmp/ps_trace.so python scripts/trace_ps.py
Softmax slots: 0 before s_full wait, 1 S ready, 2 max done, 3 chunk-a slot free,
4 chunk a published, 5 chunk-b slot free, 6 chunk b published.
MMA slots: 0 iteration start, 1 QK(j+1) issued, 2 V_j landed, 3 P.V(j) issued."""
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
t = buf.reshape(2, 20, 64, 8)[0].astype(np.int64)
print("MMA warp (median cycles over tiles 8..60): iter period, start->QK issued, ->V landed, ->PV issued")
m = t[1][8:60]
print(int(np.median(np.diff(t[1][8:61, 0]))), [int(np.median(m[:, b] - m[:, a])) for a, b in ((0, 1), (1, 2), (2, 3))])
print("softmax warps: period, wait S, S->max, max->a free, a free->a pub, a pub->b free, b free->b pub")
for w in range(4, 12):
    s = t[w][8:60]
    per = int(np.median(np.diff(t[w][8:61, 1])))
    print(w, per, [int(np.median(s[:, b] - s[:, a])) for a, b in ((0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6))])
