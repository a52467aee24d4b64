"""float64 block attention and lse merge (oracle; test infrastructure only).

Restates the reference numeric contract:

* ``attention_block``  -- ref ``_kernels_ref.py:34-54`` / ``_kernels.pyx:15-65``:
  scale 1/sqrt(D); causal key j visible iff q_off + i >= k_off + j; rows with
  no visible key give lse = -inf and a zero output row; FULL mask returns the
  identity without reading inputs.
* ``merge_state`` -- ref ``_kernels.pyx:68-102`` (the stable sign-branch form
  of ``_kernels_ref.py:57-73``): -inf rows are exact identities.

Work is done one head and one row-panel at a time so that sampled checks at
long sequence lengths do not materialise an (H, Tq, Tk) score tensor; rows
and heads are independent, so the result is the same as the batched form.
"""

import numpy as np

MASK_NONE, MASK_FULL, MASK_CAUSAL = 0, 1, 2   # ref _kernels_ref.py:27-29

_PANEL = 2048


def attention_block(q, k, v, mask_kind=MASK_NONE, q_offset=0, k_offset=0):
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    tq, heads, dim = q.shape
    tk = k.shape[0]
    out = np.zeros((tq, heads, dim))
    lse = np.full((heads, tq), -np.inf)
    if mask_kind == MASK_FULL:
        return out, lse
    scale = 1.0 / np.sqrt(dim)
    keys = k_offset + np.arange(tk)
    for h in range(heads):
        kh = np.ascontiguousarray(k[:, h, :])
        vh = np.ascontiguousarray(v[:, h, :])
        for r0 in range(0, tq, _PANEL):
            r1 = min(tq, r0 + _PANEL)
            s = (q[r0:r1, h, :] @ kh.T) * scale
            if mask_kind == MASK_CAUSAL:
                rows = q_offset + np.arange(r0, r1)
                s[rows[:, None] < keys[None, :]] = -np.inf
            m = s.max(axis=1)
            alive = np.isfinite(m)
            shift = np.where(alive, m, 0.0)
            w = np.exp(s - shift[:, None])
            tot = w.sum(axis=1)
            safe = np.where(alive, tot, 1.0)
            lse[h, r0:r1] = np.where(alive, shift + np.log(safe), -np.inf)
            out[r0:r1, h, :] = (w / safe[:, None]) @ vh
    return out, lse


def merge_state(acc_out, acc_lse, blk_out, blk_lse):
    """Return the merged (out, lse); inputs are not modified."""
    a_out = np.asarray(acc_out, dtype=np.float64)
    b_out = np.asarray(blk_out, dtype=np.float64)
    a = np.asarray(acc_lse, dtype=np.float64)
    b = np.asarray(blk_lse, dtype=np.float64)
    a_dead = np.isneginf(a)
    b_dead = np.isneginf(b)
    live = ~(a_dead | b_dead)
    with np.errstate(invalid="ignore"):
        d = np.where(live, b - a, 0.0)
    e = np.exp(-np.abs(d))
    w = np.where(d >= 0, 1.0 / (1.0 + e), e / (1.0 + e))
    lse = np.where(d >= 0, b, a) + np.log1p(e)
    # identities: blk dead -> keep acc; acc dead -> take blk
    w = np.where(b_dead, 0.0, np.where(a_dead, 1.0, w))
    lse = np.where(b_dead, a, np.where(a_dead, b, lse))
    wt = w.T[:, :, None]
    out = a_out + wt * (b_out - a_out)
    # exact pass-through on identity rows (no a + 1*(b-a) rounding)
    out = np.where(b_dead.T[:, :, None], a_out, out)
    out = np.where((a_dead & ~b_dead).T[:, :, None], b_out, out)
    return out, lse


def dense_attention(q, k, v, causal=False):
    """ref core.py:162-181: one attention_block over the whole sequence."""
    return attention_block(q, k, v, MASK_CAUSAL if causal else MASK_NONE, 0, 0)


def max_relative_error(got_out, got_lse, ref_out, ref_lse):
    """ref core.py:184-202: norm-wise disagreement of two partials."""
    got_out = np.asarray(got_out, dtype=np.float64)
    ref_out = np.asarray(ref_out, dtype=np.float64)
    got_lse = np.asarray(got_lse, dtype=np.float64)
    ref_lse = np.asarray(ref_lse, dtype=np.float64)
    scale = np.abs(ref_out).max()
    out_err = np.abs(got_out - ref_out).max() / (scale if scale > 0 else 1.0)
    both = np.isneginf(got_lse) & np.isneginf(ref_lse)
    d = np.where(both, 0.0, got_lse - ref_lse)
    if not np.isfinite(d).all():
        return np.inf
    lscale = max(1.0, np.abs(np.where(both, 0.0, ref_lse)).max())
    return float(max(out_err, np.abs(d).max() / lscale))
