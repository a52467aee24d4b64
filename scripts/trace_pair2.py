"""TR_TRACE timeline of the CTA-pair product kernel (attn_fwd_pair2.cu),
CTA 0 (the leader): per kv tile, for each 128-row half, when S was ready,
the row max done, each P chunk published (slowest of the half's 4 warps) and
seen by the MMA warp, and the next S of that half ready.  Medians over the
steady-state tiles (clock64 of CTA 0's SM).

    python -m paper_2412_20501_b200.build -D TR_TRACE --out paper_2412_20501_b200/_variants/lib_trace_pair2.so
    TOKENRING_LIB=paper_2412_20501_b200/_variants/lib_trace_pair2.so python scripts/trace_pair2.py
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

tq, tk, h, d = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (8192, 16384, 32, 128)))
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
t_all = buf.reshape(2, 20, 64, 8).astype(np.int64)
t = t_all[0]                                           # CTA 0
J = np.arange(8, 56)
mma = t[1]
med = lambda x: float(np.median(x))  # noqa: E731
print(f"shape {tq}x{tk} H={h} D={d}; CTA 0; medians over kv tiles {J[0]}..{J[-1]} (cycles)")
print(f"MMA period (K_j landed -> K_j+1 landed): {med(np.diff(mma[8:57, 0]))}")
for half, ws, seen0, seen1 in ((0, range(4, 8), 4, 5), (1, range(8, 12), 1, 2)):
    sw = t[list(ws)]
    s_ready = sw[:, J, 1].min(0)
    s_ready_last = sw[:, J, 1].max(0)
    mx = sw[:, J, 2].max(0)
    c0 = sw[:, J, 3].max(0)
    c1 = sw[:, J, 4].max(0)
    nxt = sw[:, J + 1, 1].min(0)
    ms0, ms1 = mma[J, seen0], mma[J, seen1]
    print(f"half {half}: S ready spread over warps {med(s_ready_last - s_ready):.0f} | "
          f"S ready -> max {med(mx - s_ready):.0f} -> P c0 pub {med(c0 - mx):.0f} -> "
          f"P c1 pub {med(c1 - c0):.0f} | c0 pub -> MMA sees {med(ms0 - c0):.0f}, "
          f"c1 pub -> MMA sees {med(ms1 - c1):.0f} | MMA sees c1 -> next S ready "
          f"{med(nxt - ms1):.0f} | period {med(np.diff(sw[0, 8:57, 1])):.0f}")
    per_warp = [f"w{w}: max {med(t[w][J, 2] - t[w][J, 1]):.0f} c0 {med(t[w][J, 3] - t[w][J, 2]):.0f} "
                f"c1 {med(t[w][J, 4] - t[w][J, 3]):.0f}" for w in ws]
    print("   " + " | ".join(per_warp))
    if sw[:, J, 7].min() > 0:     # builds with the chunk-computed marks
        ex0 = sw[:, J, 7]
        print(f"   max->exp start {med(ex0.max(0) - mx):.0f} | exp c0 {med((sw[:, J, 5] - ex0).max(0)):.0f} "
              f"store+arrive c0 {med((sw[:, J, 3] - sw[:, J, 5]).max(0)):.0f} | exp c1 "
              f"{med((sw[:, J, 6] - sw[:, J, 3]).max(0)):.0f} store+arrive c1 "
              f"{med((sw[:, J, 4] - sw[:, J, 6]).max(0)):.0f}")
# overlap of the two halves' exp phases: [max done, c1 published] intervals
a0 = (t[list(range(4, 8))][:, J, 2].min(0), t[list(range(4, 8))][:, J, 4].max(0))
a1 = (t[list(range(8, 12))][:, J, 2].min(0), t[list(range(8, 12))][:, J, 4].max(0))
ov = np.maximum(0, np.minimum(a0[1], a1[1]) - np.maximum(a0[0], a1[0]))
ov2 = np.maximum(0, np.minimum(a0[1][1:], a1[1][:-1]) - np.maximum(a0[0][1:], a1[0][:-1]))
print(f"exp-phase overlap of the halves (same tile / half0 j+1 vs half1 j): {med(ov):.0f} / {med(ov2):.0f}")
# one tile's events in time order (relative to half 0's S ready of tile j0)
j0 = 20
base = t[4][j0, 1]
evs = [("MMA K_j landed (iter start)", mma[j0, 0]), ("MMA V_j landed", mma[j0, 3]),
       ("MMA QK0(j) issued", mma[j0, 7]), ("MMA QK1(j) issued", mma[j0, 6]),
       ("MMA QK0(j+1) issued", mma[j0 + 1, 7]), ("MMA PV0(j) c1 issued", t[2][j0, 0]),
       ("TMA K_j+1 load issued", t[0][j0 + 1, 0]), ("TMA V_j+1 load issued", t[0][j0 + 1, 1]),
       ("TMA K_j+2 load issued", t[0][j0 + 2, 0]), ("TMA K_j+3 load issued", t[0][j0 + 3, 0]),
       ("MMA sees P1(j-1) c0", mma[j0 - 1, 1]), ("MMA sees P1(j-1) c1", mma[j0 - 1, 2]),
       ("MMA sees P0(j) c0", mma[j0, 4]), ("MMA sees P0(j) c1", mma[j0, 5]),
       ("MMA sees P1(j) c0", mma[j0, 1]), ("MMA sees P1(j) c1", mma[j0, 2]),
       ("MMA K_j+1 landed (next iter)", mma[j0 + 1, 0])]
for w in (4, 5, 8, 9):
    evs += [(f"w{w} S ready", t[w][j0, 1]), (f"w{w} max done", t[w][j0, 2]),
            (f"w{w} c0 pub", t[w][j0, 3]), (f"w{w} c1 pub", t[w][j0, 4]),
            (f"w{w} next S ready", t[w][j0 + 1, 1])]
for name, x in sorted(evs, key=lambda e: e[1]):
    print(f"  {int(x - base):7d}  {name}")

# CTA 1 (the follower; its own SM clock): S ready -> P chunks published per half
t1 = t_all[1]
if t1[4:12, J, 1].min() > 0:
    for half, ws in ((0, range(4, 8)), (1, range(8, 12))):
        sw = t1[list(ws)]
        print(f"CTA 1 half {half}: S ready -> max {med(sw[:, J, 2].max(0) - sw[:, J, 1].min(0)):.0f} -> "
              f"c0 pub {med(sw[:, J, 3].max(0) - sw[:, J, 2].max(0)):.0f} -> c1 pub "
              f"{med(sw[:, J, 4].max(0) - sw[:, J, 3].max(0)):.0f} | S ready -> c1 pub "
              f"{med(sw[:, J, 4].max(0) - sw[:, J, 1].min(0)):.0f} (CTA 0: "
              f"{med(t[list(ws)][:, J, 4].max(0) - t[list(ws)][:, J, 1].min(0)):.0f})")
