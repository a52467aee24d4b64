"""Host logic of the fused transport (ring.fused_plan): every OUT_LSE message
of the reference's token-ring schedules is a whole step's rows, pushed by the
launch that computes it into a slot of its own at the home, and each home
chunk's final n-way merge folds exactly its remote partials.  Slots are never
reused within a forward, so the only wait is the home's final one -- no
cross-rank wait cycle is possible.  CPU only; the GPU side is
tests/test_gpu_ring_ipc.py."""

import pytest

from paper_2412_20501_b200.engine import build_token_ring, build_zigzag_token_ring
from paper_2412_20501_b200.ring import compile_rank, fused_plan

CASES = [(P, kind) for P in range(2, 9) for kind in ("zigzag", "direct", "token-ring")]


def _sched(P, kind):
    if kind == "token-ring":
        return build_token_ring(P, 32 * P, 1, 64)
    return build_zigzag_token_ring(P, 64 * P, 1, 64, route="direct" if kind == "direct" else "ring")


@pytest.mark.parametrize("P,kind", CASES)
def test_every_message_is_pushed_by_its_computing_step(P, kind):
    sched = _sched(P, kind)
    c = sched.chunks[0].tokens
    plans = {r: fused_plan(compile_rank(sched, r), c) for r in range(P)}
    sent = {}
    for r, fp in plans.items():
        prog = compile_rank(sched, r)
        for s, (k, dst, a, b) in fp.push.items():
            assert prog[k].send_out[0] == dst
            assert (b - a) == len(prog[s].q_ids) * c          # the whole step's rows
            sent[(dst, k)] = r
    got = {(r, k): src for r, fp in plans.items() for k, (src, _, _) in fp.recv.items()}
    assert sent == got                                         # pushes == receives


@pytest.mark.parametrize("P,kind", CASES)
def test_slots_and_final_merge_groups(P, kind):
    """One receive slot per message (0..n-1, step order); the final n-way merge
    of each home chunk folds exactly the messages carrying it -- one per
    (rank, step) that computes that chunk remotely in the schedule."""
    sched = _sched(P, kind)
    c = sched.chunks[0].tokens
    plans = sched.all_plans()
    for r in range(P):
        prog = compile_rank(sched, r)
        fp = fused_plan(prog, c)
        assert sorted(slot for _, _, slot in fp.recv.values()) == list(range(len(fp.recv)))
        assert [fp.slot_of(k) for k in sorted(fp.recv)] == list(range(len(fp.recv)))
        home = prog[0].q_layout
        groups = fp.merge_groups(home)
        for a in home:
            remote = len({(q, i) for q in range(P) if q != r for i, p in enumerate(plans)
                          for cp in p.computes[q] if cp.q_chunk == a})
            assert len(groups[a]) == remote, (r, a)
            for slot, j in groups[a]:
                k = sorted(fp.recv)[slot]
                assert fp.recv[k][1][j] == a
