"""Test-only device-op stand-in for the ring runner on CPU/gloo: the float64
oracle behind the same interface as ``paper_2412_20501_b200.ring.CudaOps``.
Never used by the product path."""

import numpy as np
import torch

from oracle import kernels as ok


class _Ev:
    def elapsed_time(self, other):
        return 0.0


class OracleOps:
    device = torch.device("cpu")

    def attention(self, q, k, v, q_segs, kv_segs, causal, out, lse):
        qn, kn, vn = (x.double().numpy() for x in (q, k, v))
        h, d = q.shape[1], q.shape[2]
        for r0, rows, pos in q_segs:
            acc_o = np.zeros((rows, h, d))
            acc_l = np.full((h, rows), -np.inf)
            for k0, krows, kpos in kv_segs:
                mask = ok.MASK_CAUSAL if causal else ok.MASK_NONE
                bo, bl = ok.attention_block(qn[r0:r0 + rows], kn[k0:k0 + krows],
                                            vn[k0:k0 + krows], mask, pos, kpos)
                acc_o, acc_l = ok.merge_state(acc_o, acc_l, bo, bl)
            out[r0:r0 + rows] = torch.as_tensor(acc_o, dtype=torch.float32).to(out.dtype)
            lse[:, r0:r0 + rows] = torch.as_tensor(acc_l, dtype=torch.float32)

    def merge_(self, acc_out, acc_lse, blk_out, blk_lse):
        o, l = ok.merge_state(acc_out.double().numpy(), acc_lse.double().numpy(),
                              blk_out.double().numpy(), blk_lse.double().numpy())
        acc_out.copy_(torch.as_tensor(o, dtype=torch.float32))
        acc_lse.copy_(torch.as_tensor(l, dtype=torch.float32))

    def init_(self, acc_out, acc_lse):
        acc_out.zero_()
        acc_lse.fill_(float("-inf"))

    def event(self):
        return _Ev()

    def record(self, ev):
        pass
