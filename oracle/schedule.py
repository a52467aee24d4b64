"""Schedule builders and step executor (oracle; test infrastructure only).

Restates ``pkg/src/ringsim/engine.py``.  A schedule is kept in the canonical
plain form that ``scripts/make_golden.py`` also dumps the reference's
``Schedule`` objects into, so that oracle, product and reference schedules
compare with ``==``:

    {"kind", "ranks", "causal", "chunks": [[id, start, stop, home], ...],
     "steps": [plan, ...], "final": plan | None}
    plan = [per-rank {"computes": [[q, kv, mask, q_off, k_off, acc], ...],
                      "sends":    [[dst, kind, [chunk ids], elements], ...],
                      "merges":   [[src, [chunk ids]], ...]}]

``mask`` is "none" | "fully_masked" | "causal"; ``kind`` is "q_block" |
"kv_block" | "out_lse".
"""

import numpy as np

from . import partition as part
from .kernels import MASK_CAUSAL, MASK_FULL, MASK_NONE, attention_block, merge_state


def _plan(p):
    return [{"computes": [], "sends": [], "merges": []} for _ in range(p)]


def _q_el(t, h, d):          # ref engine.py:147-148
    return t * h * d


def _kv_el(t, h, d):         # ref engine.py:151-152
    return 2 * t * h * d


def _out_el(t, h, d):        # ref engine.py:155-157
    return t * h * d + h * t


def _trivial(kind, seq_len, causal):     # ref engine.py:176-184
    plan = _plan(1)
    plan[0]["computes"].append([0, 0, "causal" if causal else "none", 0, 0, True])
    return {"kind": kind, "ranks": 1, "causal": causal,
            "chunks": [[0, 0, seq_len, 0]], "steps": [plan], "final": None}


def _wire_merges(s):         # ref engine.py:187-200
    plans = s["steps"] + ([s["final"]] if s["final"] is not None else [])
    for i in range(len(plans) - 1):
        for r in range(s["ranks"]):
            for dst, kind, ids, _ in plans[i][r]["sends"]:
                if kind == "out_lse":
                    plans[i + 1][dst]["merges"].append([r, list(ids)])
    return s


def ring(p, seq_len, h, d, causal=False):           # ref engine.py:203-230
    part.contiguous(seq_len, p)
    if p == 1:
        return _trivial("ring", seq_len, causal)
    n = seq_len // p
    chunks = [[r, r * n, (r + 1) * n, r] for r in range(p)]
    steps = []
    for i in range(p):
        plan = _plan(p)
        for j in range(p):
            b = (j - i) % p
            if not causal or j > b:
                m = ["none", 0, 0]
            elif j == b:
                m = ["causal", chunks[j][1], chunks[b][1]]
            else:
                m = ["fully_masked", 0, 0]
            plan[j]["computes"].append([j, b, m[0], m[1], m[2], True])
            if i < p - 1:
                plan[j]["sends"].append([(j + 1) % p, "kv_block", [b], _kv_el(n, h, d)])
        steps.append(plan)
    return {"kind": "ring", "ranks": p, "causal": causal, "chunks": chunks,
            "steps": steps, "final": None}


def node_ring(kind, nodes, g, seq_len, h, d):      # ref engine.py:233-290
    """Token ring inside each node of g ranks, KV hand-off across nodes."""
    p = nodes * g
    part.contiguous(seq_len, p)
    if p == 1:
        return _trivial(kind, seq_len, False)
    n = seq_len // p
    chunks = [[r, r * n, (r + 1) * n, r] for r in range(p)]
    steps, final = [], None
    for ph in range(nodes):
        s0 = ph % g
        for s in range(g):
            plan = _plan(p)
            for m in range(nodes):
                for loc in range(g):
                    r = m * g + loc
                    resident = m * g + (loc + ph - s) % g
                    kv = ((m - ph) % nodes) * g + loc
                    plan[r]["computes"].append([resident, kv, "none", 0, 0, s == s0])
                    if s < g - 1:
                        plan[r]["sends"].append([m * g + (loc + 1) % g, "q_block", [resident],
                                                 _q_el(n, h, d)])
                    if s >= 1 and (s - 1) != s0:
                        prev = m * g + (loc + ph - (s - 1)) % g
                        plan[r]["sends"].append([prev, "out_lse", [prev], _out_el(n, h, d)])
            steps.append(plan)
        ret = _plan(p)
        for m in range(nodes):
            for loc in range(g):
                r = m * g + loc
                if (g - 1) != s0:
                    prev = m * g + (loc + ph - (g - 1)) % g
                    ret[r]["sends"].append([prev, "out_lse", [prev], _out_el(n, h, d)])
                if ph < nodes - 1:
                    kv = ((m - ph) % nodes) * g + loc
                    ret[r]["sends"].append([((m + 1) % nodes) * g + loc, "kv_block", [kv],
                                            _kv_el(n, h, d)])
        if ph < nodes - 1:
            steps.append(ret)
        else:
            final = ret
    return _wire_merges({"kind": kind, "ranks": p, "causal": False, "chunks": chunks,
                         "steps": steps, "final": final})


def token_ring(p, seq_len, h, d):                   # ref engine.py:293-295
    return node_ring("token-ring", 1, p, seq_len, h, d)


def hybrid(nodes, g, seq_len, h, d):                # ref engine.py:298-303
    return node_ring("hybrid", nodes, g, seq_len, h, d)


def zigzag_token_ring(p, seq_len, h, d):            # ref engine.py:306-366
    part.zigzag(seq_len, p)
    if p == 1:
        return _trivial("zigzag-token-ring", seq_len, True)
    c = seq_len // (2 * p)
    chunks = [[a, a * c, (a + 1) * c, min(a, 2 * p - 1 - a)] for a in range(2 * p)]
    alive = {o: [o, 2 * p - 1 - o] for o in range(p)}
    prev_done = {}
    steps, final = [], None
    for i in range(p + 1):
        plan = _plan(p)
        done_now = {}
        for r in range(p):
            if i < p:
                o = (r - i) % p
                mine = (r, 2 * p - 1 - r)
                done = []
                for a in alive[o]:
                    hit = False
                    for b in mine:
                        if a > b:
                            plan[r]["computes"].append([a, b, "none", 0, 0, i == 0])
                            hit = True
                        elif a == b:
                            plan[r]["computes"].append(
                                [a, b, "causal", a * c, b * c, i == 0])
                            hit = True
                    if hit:
                        done.append(a)
                done_now[r] = done
                if i < p - 1:
                    hosts = [(o + s) % p for s in range(i + 1, p)]
                    keep = [a for a in alive[o] if any(a >= x for x in hosts)]
                    alive[o] = keep
                    plan[r]["sends"].append(
                        [(r + 1) % p, "q_block", list(keep), _q_el(len(keep) * c, h, d)])
            if i >= 2:
                ids = prev_done[r]
                plan[r]["sends"].append(
                    [(r - i + 1) % p, "out_lse", list(ids), len(ids) * _out_el(c, h, d)])
        if i < p:
            prev_done = done_now
            steps.append(plan)
        else:
            final = plan
    return _wire_merges({"kind": "zigzag-token-ring", "ranks": p, "causal": True,
                         "chunks": chunks, "steps": steps, "final": final})


def by_name(kind, p, seq_len, h, d, causal=False, nodes=1):
    """Builder by the reference CLI's schedule names (ref cli.py:167-180)."""
    if kind == "ring":
        return ring(p, seq_len, h, d, causal)
    if kind == "token-ring":
        return token_ring(p, seq_len, h, d)
    if kind == "hybrid":
        return hybrid(nodes, p // nodes, seq_len, h, d)
    if kind == "zigzag-token-ring":
        return zigzag_token_ring(p, seq_len, h, d)
    raise ValueError(kind)


def ranges_of(sched, seq_len):
    if sched["kind"] == "zigzag-token-ring":
        return part.zigzag(seq_len, sched["ranks"])
    return part.contiguous(seq_len, sched["ranks"])


_MASK = {"none": MASK_NONE, "fully_masked": MASK_FULL, "causal": MASK_CAUSAL}


def execute(sched, q, k, v, attn=attention_block, merge=merge_state):
    """Step-barrier execution over simulated ranks (ref engine.py:468-638).

    Returns per-rank (out, lse) over the rank's home chunks in start order.
    ``attn``/``merge`` default to the float64 oracle kernels.
    """
    heads, dim = q.shape[1], q.shape[2]
    ch = {c[0]: c for c in sched["chunks"]}
    qs = {r: {} for r in range(sched["ranks"])}
    kvs = {r: {} for r in range(sched["ranks"])}
    for cid, a, b, home in sched["chunks"]:
        qs[home][cid] = q[a:b]
        kvs[home][cid] = (k[a:b], v[a:b])
    acc = {cid: (np.zeros((b - a, heads, dim)), np.full((heads, b - a), -np.inf))
           for cid, a, b, _ in sched["chunks"]}
    stash = {r: None for r in range(sched["ranks"])}
    flight = []
    plans = sched["steps"] + ([sched["final"]] if sched["final"] is not None else [])

    def fold(msg):
        for cid in msg[3]:
            acc[cid] = merge(acc[cid][0], acc[cid][1], *msg[4][cid])

    for plan in plans:
        arrivals, flight = flight, []
        for msg in arrivals:                     # (src, dst, kind, ids, payload)
            if msg[2] == "q_block":
                for cid, blk in zip(msg[3], msg[4]):
                    qs[msg[1]][cid] = blk
            elif msg[2] == "kv_block":
                kvs[msg[1]][msg[3][0]] = msg[4]
        for msg in arrivals:
            if msg[2] == "out_lse":
                fold(msg)
        outgoing = {}
        for r in range(sched["ranks"]):
            for dst, kind, ids, _ in plan[r]["sends"]:
                if kind == "out_lse":
                    outgoing[r] = stash[r]
                    stash[r] = None
        for r in range(sched["ranks"]):
            res, accumulate = {}, None
            for a, b, m, qo, ko, accu in plan[r]["computes"]:
                kb, vb = kvs[r][b]
                blk = attn(qs[r][a], kb, vb, _MASK[m], qo, ko)
                res[a] = merge(*res[a], *blk) if a in res else blk
                accumulate = accu
            if res:
                if accumulate:
                    for a in sorted(res):
                        acc[a] = merge(acc[a][0], acc[a][1], *res[a])
                else:
                    stash[r] = res
        for r in range(sched["ranks"]):
            for dst, kind, ids, _ in plan[r]["sends"]:
                if kind == "q_block":
                    flight.append((r, dst, kind, ids, [qs[r].pop(x) for x in ids]))
                elif kind == "kv_block":
                    flight.append((r, dst, kind, ids, kvs[r].pop(ids[0])))
                else:
                    flight.append((r, dst, kind, ids, outgoing[r]))
    for msg in flight:
        fold(msg)
    outs = {}
    for r in range(sched["ranks"]):
        owned = sorted((c for c in sched["chunks"] if c[3] == r), key=lambda c: c[1])
        outs[r] = (np.concatenate([acc[c[0]][0] for c in owned], axis=0),
                   np.concatenate([acc[c[0]][1] for c in owned], axis=1))
    return outs


def flops(sched, heads, dim):
    """Algorithmic flops 4*H*D*(unmasked pairs) (ref engine.py:160-173)."""
    ch = {c[0]: c for c in sched["chunks"]}
    total = 0
    plans = sched["steps"] + ([sched["final"]] if sched["final"] is not None else [])
    for plan in plans:
        for r in range(sched["ranks"]):
            for a, b, m, qo, ko, _ in plan[r]["computes"]:
                tq = ch[a][2] - ch[a][1]
                tk = ch[b][2] - ch[b][1]
                if m == "none":
                    pairs = tq * tk
                elif m == "fully_masked":
                    pairs = 0
                else:
                    pairs = int(np.clip(qo + np.arange(tq) - ko + 1, 0, tk).sum())
                total += 4 * heads * dim * pairs
    return total
