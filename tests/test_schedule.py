"""The product's schedule compiler and partitions vs the reference's own
objects (tests/golden/schedules.json, dumped from ringsim) -- bit-exact.
CPU only."""

import numpy as np
import pytest

from paper_2412_20501_b200 import engine, partition
from paper_2412_20501_b200.core import MaskSpec
from paper_2412_20501_b200.errors import ConfigError


def canon(s):
    def plan(p):
        return [{
            "computes": [[cp.q_chunk, cp.kv_chunk, cp.mask.kind.value, int(cp.mask.q_offset),
                          int(cp.mask.k_offset), bool(cp.accumulate)] for cp in p.computes[r]],
            "sends": [[m.dst, m.kind.value, list(m.chunk_ids), int(m.payload_elements)]
                      for m in p.sends[r]],
            "merges": [[mp.src, list(mp.chunk_ids)] for mp in p.merges[r]],
        } for r in range(s.ranks)]
    return {"kind": s.kind, "ranks": s.ranks, "causal": bool(s.causal),
            "chunks": [[c.id, c.start, c.stop, c.home] for c in s.chunks],
            "steps": [plan(p) for p in s.steps],
            "final": plan(s.final_phase) if s.final_phase else None}


def build(kind, p, s, h, d, causal, nodes=1):
    return engine.build_schedule(kind, p, s, h, d, causal if kind == "ring" else None,
                                 nodes=nodes)


def test_schedules_bit_exact(golden_schedules):
    for g in golden_schedules:
        kind, p, s, h, d, causal = g["args"][:6]
        sc = build(*g["args"])
        assert canon(sc) == g["schedule"], g["args"]
        assert [list(map(list, sc.partition.ranges(r))) for r in range(p)] == g["ranges"]
        assert list(partition.causal_work_count(sc.partition)) == g["causal_work"]
        tr = engine.trace_from_schedule(sc)
        assert sum(c.flops for c in tr.computes) == g["flops_total"]
        assert [[c.step, c.rank, c.flops] for c in tr.computes] == g["flops_per_step_rank"]
        vol = engine.comm_volume(sc)
        got = sorted([[st, r, k.value, n] for (st, r, k), n in vol.entries.items()],
                     key=lambda x: (x[0], x[1], x[2]))
        assert got == g["volume"], g["args"]


def test_unmasked_pairs_closed_form():
    rng = np.random.default_rng(0)
    for _ in range(500):
        tq, tk = rng.integers(1, 40, 2)
        qo, ko = rng.integers(0, 60, 2)
        m = MaskSpec.causal(int(qo), int(ko))
        brute = int(np.clip(qo + np.arange(tq) - ko + 1, 0, tk).sum())
        assert engine.unmasked_pairs(m, int(tq), int(tk)) == brute


def test_config_volumes_and_flops():
    # ref tests/test_engine.py:288-331 and BASELINE.md
    tr = engine.build_token_ring(4, 24000, 32, 128)
    vol = engine.comm_volume(tr)
    assert vol.forward_elements(step=1, rank=0) * 2 == 49_152_000
    assert vol.reverse_elements(step=2, rank=0) * 2 == 49_536_000
    ring = engine.build_ring_attention(4, 24000, 32, 128)
    assert engine.comm_volume(ring).forward_elements(step=0, rank=0) * 2 == 98_304_000
    zz = engine.build_zigzag_token_ring(8, 131072, 32, 128)
    S = 131072
    # 1.407386e14 algorithmic flops for config 3
    assert engine.total_flops(zz) == 4 * 32 * 128 * (S * (S + 1) // 2) == 140738562097152


def test_zigzag_partition_rules():
    p = partition.split_zigzag(16, 4)
    assert p.ranges(0) == ((0, 2), (14, 16))
    assert p.ranges(3) == ((6, 8), (8, 10))
    assert partition.causal_work_count(p) == (34, 34, 34, 34)
    p.validate()
    with pytest.raises(ConfigError):
        partition.split_zigzag(18, 4)
    with pytest.raises(ConfigError):
        partition.split_contiguous(10, 4)
    assert p.local_offset(1, 12) == 2


def test_gather_and_reorder_roundtrip_numpy():
    p = partition.split_zigzag(32, 4)
    x = np.arange(32 * 2 * 3).reshape(32, 2, 3)
    parts = [partition.gather_local(x, p, r) for r in range(4)]
    back = np.empty_like(x)
    for r in range(4):
        cur = 0
        for a, b in p.ranges(r):
            back[a:b] = parts[r][cur:cur + b - a]
            cur += b - a
    assert np.array_equal(back, x)


def test_rank_programs_cover_all_pairs_once():
    """Every causal (q chunk, kv chunk) pair is computed exactly once across
    ranks and steps, and every rank does identical work each step."""
    from paper_2412_20501_b200.ring import compile_rank
    for P in (2, 3, 4, 8):
        sc = engine.build_zigzag_token_ring(P, 32 * P, 1, 4)
        seen = {}
        for r in range(P):
            for st in compile_rank(sc, r):
                for a in st.q_ids:
                    for b in st.kv_ids:
                        if a >= b:
                            seen[(a, b)] = seen.get((a, b), 0) + 1
        want = {(a, b) for a in range(2 * P) for b in range(2 * P) if a >= b}
        assert set(seen) == want and all(v == 1 for v in seen.values())


@pytest.mark.parametrize("P", [2, 3, 4, 5, 8])
def test_direct_route_same_computes_fewer_q_bytes(P):
    """NVSwitch-aware Q routing (a non-reference schedule):
    identical computes and merges at every rank and step, Q chunk-hops
    reduced from (P-1)(2P-1) to (P-1)(2P-1) - (P-1)(P-2)/2, and every
    compiled rank program still finds each q chunk it computes or forwards."""
    from paper_2412_20501_b200.ring import compile_rank
    c, H, D = 16, 2, 8
    ref = engine.build_zigzag_token_ring(P, 2 * P * c, H, D)
    dr = engine.build_schedule("zigzag-token-ring-direct", P, 2 * P * c, H, D)
    assert dr.kind == "zigzag-token-ring-direct" and dr.n_steps == ref.n_steps
    for a, b in zip(ref.all_plans(), dr.all_plans()):
        assert a.computes == b.computes and a.merges == b.merges
        for r in range(P):
            assert ([m for m in a.sends[r] if m.kind is engine.MsgKind.OUT_LSE]
                    == [m for m in b.sends[r] if m.kind is engine.MsgKind.OUT_LSE])

    def q_hops(s):
        return sum(n for (_, _, k), n in engine.comm_volume(s).entries.items()
                   if k is engine.MsgKind.Q_BLOCK) // (c * H * D)
    assert q_hops(ref) == (P - 1) * (2 * P - 1)
    assert q_hops(dr) == (P - 1) * (2 * P - 1) - (P - 1) * (P - 2) // 2
    for r in range(P):
        compile_rank(dr, r)
    if P == 2:
        assert canon(dr)["steps"] == canon(ref)["steps"]
    with pytest.raises(ConfigError):
        engine.build_zigzag_token_ring(P, 2 * P * c, H, D, route="mesh")
