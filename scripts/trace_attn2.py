"""Per-tile event offsets of CTA 0 of the product kernel (TR_TRACE build).

Build:  python -m paper_2412_20501_b200.build -D TR_TRACE --out paper_2412_20501_b200/_variants/lib_trace.so
Run:    TOKENRING_LIB=paper_2412_20501_b200/_variants/lib_trace.so python scripts/trace_attn2.py

Events (clock64, all warps of CTA 0 share one SM clock), medians over kv
tiles 8..56 of a full 8192x16384 launch, relative to the MMA warp seeing K_j:
  MMA  0 K_j ready   1 S0=Q0.K_j issued   2 P1(j-1) seen, O1 += P1.V(j-1) issued
       3 S1=Q1.K_j issued, V_j ready       4 P0(j) seen, O0 += P0.V_j issued
  softmax warp (half h)  0 wait for S_h(j) starts  1 S_h(j) ready  2 max done
       3 P_h(j) published; 4/5 first P chunk computed / published, 6/7 second
"""
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
CTA = int(os.environ.get("CTA", "0"))      # 1: the second CTA of a pair build
buf = np.zeros(2 * 20 * 64 * 8, dtype=np.uint64)
L = _lib.lib()
fn = getattr(L, os.environ.get("TRACE_SYM", "tr_debug_trace"))   # tr_debug_trace_pair2: pair build
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert fn(buf.ctypes.data, buf.nbytes) == 0
t_all = buf.reshape(2, 20, 64, 8).astype(np.int64)
t = t_all[CTA]
if CTA:   # softmax events of CTA 1 against the leader's MMA warp (cluster-local clocks differ)
    t = t.copy()
    t[1] = t_all[0][1]
J = slice(8, 56)
base = t[1, J, 0]
period = np.median(np.diff(t[1, 8:57, 0]))
print(f"kv-tile period (MMA warp): {period:.0f} cycles (tensor work 2048)")
print("MMA warp events vs K_j ready:", [int(np.median(t[1, J, s] - base)) for s in range(5)])
for w in range(4, 12):
    print(f"softmax warp {w} (half {(w - 4) // 4}, SMSP {w % 4}):",
          [int(np.median(t[w, J, s] - base)) for s in range(4)],
          " S ready->max", int(np.median(t[w, J, 2] - t[w, J, 1])),
          " max->P", int(np.median(t[w, J, 3] - t[w, J, 2])),
          " | chunk0 exp", int(np.median(t[w, J, 4] - t[w, J, 2])),
          " store+arrive", int(np.median(t[w, J, 5] - t[w, J, 4])),
          " chunk1 exp", int(np.median(t[w, J, 6] - t[w, J, 5])),
          " store+arrive", int(np.median(t[w, J, 7] - t[w, J, 6])))
# per-half: the slowest quarter decides P publication
for hh in (0, 1):
    last = np.max(t[4 + 4 * hh:8 + 4 * hh, J, 3], axis=0)
    first_ready = np.min(t[4 + 4 * hh:8 + 4 * hh, J, 1], axis=0)
    print(f"half {hh}: S ready (first warp) -> P published (last warp) median "
          f"{int(np.median(last - first_ready))}")
