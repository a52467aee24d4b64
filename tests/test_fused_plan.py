"""Host logic of the fused transport (ring.fused_plan): every OUT_LSE message
of the reference's token-ring schedules is a whole step's rows, each receive
slot is granted exactly once per message and only after the previous
message in it was merged, and the protocol (waits on o_ready / grant flags,
in each rank's program order) runs to completion for every rank count.
CPU only; the GPU side is tests/test_gpu_ring_ipc.py."""

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
def test_grants_cover_each_message_once_and_follow_slot_reuse(P, kind):
    sched = _sched(P, kind)
    c = sched.chunks[0].tokens
    for r in range(P):
        fp = fused_plan(compile_rank(sched, r), c)
        granted = [k for _, k in fp.grant_at_start] + [k2 for _, k2 in fp.grant_after.values()]
        assert sorted(granted) == sorted(fp.recv)
        for k, (src, k2) in fp.grant_after.items():
            assert fp.recv[k][2] == fp.recv[k2][2] and k < k2      # same slot, later message
            assert fp.recv[k2][0] == src
            # the slot is still in use by k until it is merged (step k+1), and
            # no other message lands in it in between
            assert not any(fp.recv[j][2] == fp.recv[k][2] for j in fp.recv if k < j < k2)


@pytest.mark.parametrize("P,kind", CASES)
def test_protocol_runs_to_completion(P, kind):
    """Discrete simulation of the flag protocol of ring._forward_ipc (fused):
    per rank, step i waits for o_ready(msg i-1), merges it (raising the next
    grant into that slot), then -- if it pushes -- waits for its own grant
    and computes (raising the home's o_ready).  Must not deadlock."""
    sched = _sched(P, kind)
    c = sched.chunks[0].tokens
    progs = {r: compile_rank(sched, r) for r in range(P)}
    fps = {r: fused_plan(progs[r], c) for r in range(P)}
    o_ready, grant = set(), set()             # (home, k), (sender, k)
    for r in range(P):
        for src, k in fps[r].grant_at_start:
            grant.add((src, k))
    pc = {r: (0, 0) for r in range(P)}        # (step, phase): phase 0 = merge, 1 = compute
    n = len(progs[0])
    progressed = True
    while progressed:
        progressed = False
        for r in range(P):
            (i, ph), fp = pc[r], fps[r]
            if i >= n:
                continue
            if ph == 0:
                if i >= 1 and (i - 1) in fp.recv:
                    if (r, i - 1) not in o_ready:
                        continue
                    if (i - 1) in fp.grant_after:
                        grant.add(fp.grant_after[i - 1])
                pc[r] = (i, 1)
            else:
                if i in fp.push:
                    k, dst, _, _ = fp.push[i]
                    if (r, k) not in grant:
                        continue
                    assert (dst, k) not in o_ready
                    o_ready.add((dst, k))
                pc[r] = (i + 1, 0)
            progressed = True
    for r in range(P):                        # the final merge after the loop
        last = n - 1
        assert last not in fps[r].recv or (r, last) in o_ready
    assert all(v == (n, 0) for v in pc.values()), pc
