"""Small launches of every product kernel for compute-sanitizer
(memcheck / racecheck / synccheck): the CTA-pair tcgen05 kernel (plain,
causal with a diagonal, multi-segment, float32 out, push with done flag), the
single-CTA D=64 kernel, the CUDA-core kernel, the pairwise and n-way merges,
SplitMix64, partial init and the flag kernels.  Used by scripts/sanitize.sh."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20501_b200 import kernels as K  # noqa: E402

torch.manual_seed(0)


def r(*s):
    return (torch.randn(*s, device="cuda") * 0.5).to(torch.bfloat16)


for tq, tk, h, d, mask in [(512, 1024, 2, 128, 0), (640, 640, 2, 128, 2), (256, 384, 2, 64, 2),
                           (100, 90, 2, 32, 2)]:
    q, k, v = r(tq, h, d), r(tk, h, d), r(tk, h, d)
    K.attention_block(q, k, v, mask, 0, 0)
c, h, d = 512, 2, 128
q, k, v = r(2 * c, h, d), r(2 * c, h, d), r(2 * c, h, d)
segs = [(0, c, 0), (c, c, 3 * c)]
acc = torch.empty(2 * c, h, d, device="cuda")
lse = torch.empty(h, 2 * c, device="cuda")
K.attention_segments(q, k, v, segs, segs, True, acc, lse)            # float32 out
ob = torch.empty(c, h, d, dtype=torch.bfloat16, device="cuda")
lb = torch.empty(h, c, device="cuda")
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
flag = torch.zeros(1, dtype=torch.int64, device="cuda")
K.attention_segments_push(q, k, v, [(c, c, 3 * c)], segs, True, ob, lb, c, cnt, flag, 7)
K.flag_wait_(flag, 7)
K.merge_state_(acc[:c], lse[:, :c], ob, lb)
K.merge_n_(acc[c:], lse[:, c:], [(ob, lb), (ob, lb), (ob, lb)])
K.partial_init_(acc, lse)
K.splitmix_bf16_(q, 3, 0)
torch.cuda.synchronize()
K.poll_error()
print("sanitize_small ok")
