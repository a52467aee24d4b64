"""Schedules (ring, token ring, zigzag token ring) and the single-device
executor.

The schedule IR keeps the reference's types and field names
(``pkg/src/ringsim/engine.py:59-144``) so code written against
``ringsim.engine`` reads the same.  The builders are a per-rank *step-program
compiler*: each rank's sends / computes / merges at step i are produced from
closed forms rather than by simulating the traveling sets,
and tests/test_schedule.py checks the result field-by-field against the
reference's own ``Schedule`` objects (tests/golden/schedules.json).

``execute`` runs a schedule with every simulated rank on one GPU: blocks live
in global device buffers, a "send" hands a buffer view over, and every
rank's computes of one step go to the sm_100a kernel as ONE segmented launch
(all q chunks x all kv chunks, causal by global position).  The multi-GPU
runner is ``paper_2412_20501_b200.ring``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import torch

from . import kernels
from .core import MaskKind, MaskSpec, Partial, check_qkv
from .errors import ConfigError, DimensionError, ScheduleError
from .partition import Partition, split_contiguous, split_zigzag


class MsgKind(Enum):
    Q_BLOCK = "q_block"
    KV_BLOCK = "kv_block"
    OUT_LSE = "out_lse"


FORWARD_KINDS = (MsgKind.Q_BLOCK, MsgKind.KV_BLOCK)


@dataclass(frozen=True)
class Chunk:
    id: int
    start: int
    stop: int
    home: int

    @property
    def tokens(self) -> int:
        return self.stop - self.start


@dataclass(frozen=True)
class MsgPlan:
    src: int
    dst: int
    kind: MsgKind
    chunk_ids: tuple
    payload_elements: int


@dataclass(frozen=True)
class ComputePlan:
    q_chunk: int
    kv_chunk: int
    mask: MaskSpec
    accumulate: bool


@dataclass(frozen=True)
class MergePlan:
    src: int
    chunk_ids: tuple


@dataclass
class StepPlan:
    sends: dict
    computes: dict
    merges: dict

    @classmethod
    def empty(cls, ranks: int) -> "StepPlan":
        return cls({r: [] for r in range(ranks)}, {r: [] for r in range(ranks)},
                   {r: [] for r in range(ranks)})


@dataclass
class Schedule:
    kind: str
    ranks: int
    heads: int
    head_dim: int
    causal: bool
    partition: Partition
    chunks: tuple
    steps: list
    final_phase: StepPlan | None

    @property
    def n_steps(self) -> int:
        return len(self.steps) + (1 if self.final_phase is not None else 0)

    def all_plans(self) -> list:
        return list(self.steps) + ([self.final_phase] if self.final_phase is not None else [])

    def chunk(self, cid: int) -> Chunk:
        return self.chunks[cid]


# ----------------------------------------------------------------- payloads
def q_elements(tokens, heads, head_dim):          # ref engine.py:147-148
    return tokens * heads * head_dim


def kv_elements(tokens, heads, head_dim):         # ref engine.py:151-152
    return 2 * tokens * heads * head_dim


def out_lse_elements(tokens, heads, head_dim):    # ref engine.py:155-157
    return tokens * heads * head_dim + heads * tokens


def unmasked_pairs(mask: MaskSpec, tq: int, tk: int) -> int:
    """Score pairs a masked block computes (ref engine.py:160-167), closed form."""
    if mask.kind == MaskKind.NONE:
        return tq * tk
    if mask.kind == MaskKind.FULLY_MASKED:
        return 0
    # visible(i) = clip(q_off + i - k_off + 1, 0, tk), summed over i in [0, tq)
    base = mask.q_offset - mask.k_offset + 1
    total = 0
    lo = max(0, -base)                 # first i with visible > 0
    hi = min(tq, tk - base)            # first i with visible == tk
    if hi > lo:
        n = hi - lo
        total += n * base + (lo + hi - 1) * n // 2
    full_from = max(lo, hi, 0)
    if full_from < tq:
        total += (tq - max(full_from, 0)) * tk
    return total


def compute_flops(mask: MaskSpec, tq: int, tk: int, heads: int, head_dim: int) -> int:
    return 4 * heads * head_dim * unmasked_pairs(mask, tq, tk)


# ----------------------------------------------------------------- builders
def _trivial(kind, part, heads, head_dim, causal):
    step = StepPlan.empty(1)
    mask = MaskSpec.causal(0, 0) if causal else MaskSpec.none()
    step.computes[0].append(ComputePlan(0, 0, mask, True))
    return Schedule(kind, 1, heads, head_dim, causal, part,
                    (Chunk(0, 0, part.seq_len, 0),), [step], None)


def _wire_merges(sched: Schedule) -> Schedule:
    plans = sched.all_plans()
    for nxt, plan in zip(plans[1:], plans[:-1]):
        for r in range(sched.ranks):
            for m in plan.sends[r]:
                if m.kind is MsgKind.OUT_LSE:
                    nxt.merges[m.dst].append(MergePlan(m.src, m.chunk_ids))
    return sched


def build_ring_attention(ranks, seq_len, heads, head_dim, causal=False) -> Schedule:
    """KV rotation baseline (ref engine.py:203-230): rank j computes its own q
    against kv chunk (j-i) mod P at step i and forwards the kv block."""
    part = split_contiguous(seq_len, ranks)
    if ranks == 1:
        return _trivial("ring", part, heads, head_dim, causal)
    n = seq_len // ranks
    chunks = tuple(Chunk(r, r * n, (r + 1) * n, r) for r in range(ranks))
    steps = []
    for i in range(ranks):
        plan = StepPlan.empty(ranks)
        for j in range(ranks):
            b = (j - i) % ranks
            if not causal or j > b:
                mask = MaskSpec.none()
            elif j == b:
                mask = MaskSpec.causal(chunks[j].start, chunks[b].start)
            else:
                mask = MaskSpec.fully_masked()
            plan.computes[j].append(ComputePlan(j, b, mask, True))
            if i < ranks - 1:
                plan.sends[j].append(MsgPlan(j, (j + 1) % ranks, MsgKind.KV_BLOCK, (b,),
                                             kv_elements(n, heads, head_dim)))
        steps.append(plan)
    return Schedule("ring", ranks, heads, head_dim, causal, part, chunks, steps, None)


def _node_ring(kind, nodes, per_node, seq_len, heads, head_dim) -> Schedule:
    """TokenRing inside each node of ``per_node`` ranks, KV rotation across
    ``nodes`` nodes (ref engine.py:233-290; nodes=1 is the plain TokenRing).

    Phase p (one per node hop) has ``per_node`` steps.  Rank r = m*G + l holds
    kv chunk ((m-p) mod M)*G + l during phase p; the q chunk resident at step
    s is m*G + (l+p-s) mod G, so the rank meets its own q chunk (and
    accumulates locally) at s0 = p mod G.  Every other step's rows go back to
    the q chunk's home one step later.  Between phases a step with no
    computes returns the last rows and hands kv chunks to the next node."""
    M, G = nodes, per_node
    P = M * G
    part = split_contiguous(seq_len, P)
    if P == 1:
        return _trivial(kind, part, heads, head_dim, False)
    n = seq_len // P
    chunks = tuple(Chunk(r, r * n, (r + 1) * n, r) for r in range(P))
    qe, ke = q_elements(n, heads, head_dim), kv_elements(n, heads, head_dim)
    oe = out_lse_elements(n, heads, head_dim)
    steps, final = [], None
    for p in range(M):
        s0 = p % G
        for s in range(G):
            plan = StepPlan.empty(P)
            for r in range(P):
                m, l = divmod(r, G)
                resident = m * G + (l + p - s) % G
                plan.computes[r].append(ComputePlan(resident, ((m - p) % M) * G + l,
                                                    MaskSpec.none(), s == s0))
                if s < G - 1:
                    plan.sends[r].append(MsgPlan(r, m * G + (l + 1) % G, MsgKind.Q_BLOCK,
                                                 (resident,), qe))
                if s >= 1 and s - 1 != s0:
                    prev = m * G + (l + p - s + 1) % G
                    plan.sends[r].append(MsgPlan(r, prev, MsgKind.OUT_LSE, (prev,), oe))
            steps.append(plan)
        hand = StepPlan.empty(P)
        for r in range(P):
            m, l = divmod(r, G)
            if G - 1 != s0:
                prev = m * G + (l + p - G + 1) % G
                hand.sends[r].append(MsgPlan(r, prev, MsgKind.OUT_LSE, (prev,), oe))
            if p < M - 1:
                hand.sends[r].append(MsgPlan(r, ((m + 1) % M) * G + l, MsgKind.KV_BLOCK,
                                             (((m - p) % M) * G + l,), ke))
        if p < M - 1:
            steps.append(hand)
        else:
            final = hand
    return _wire_merges(Schedule(kind, P, heads, head_dim, False, part, chunks, steps, final))


def build_token_ring(ranks, seq_len, heads, head_dim) -> Schedule:
    """Non-causal TokenRing (ref engine.py:293-295): q chunk (r-s) mod P
    visits rank r at step s; results return to the chunk's home."""
    return _node_ring("token-ring", 1, ranks, seq_len, heads, head_dim)


def build_hybrid(nodes, ranks_per_node, seq_len, heads, head_dim) -> Schedule:
    """TokenRing inside each node, KV rotation across nodes, non-causal
    (ref engine.py:298-303)."""
    if nodes < 1 or ranks_per_node < 1:
        raise ConfigError("nodes and ranks_per_node must be >= 1")
    return _node_ring("hybrid", nodes, ranks_per_node, seq_len, heads, head_dim)


def zigzag_alive(ranks: int, origin: int, step: int) -> tuple:
    """Sub-chunks of origin ``origin`` resident on their host at ``step``.

    The high chunk 2P-1-o is needed by every host; the low chunk o is needed
    again after the ring wraps (hosts 0..o-1) unless o == 0, so chunk 0 is
    the only one ever pruned, right after step 0 (finding 3)."""
    high = 2 * ranks - 1 - origin
    return (origin, high) if (origin >= 1 or step == 0) else (high,)


def _direct_carries_low(P: int, origin: int, sender: int) -> bool:
    """Direct routing: does the ring hop sender -> sender+1 carry origin's low chunk?

    The low chunk ``origin`` is computed only at its origin (step 0) and at
    hosts 0..origin-1 (after the wrap), so on a full mesh it goes straight
    from its origin to host 0 and rides the ring only for hops 0 -> 1 -> ...
    -> origin-1, i.e. from senders 0..origin-2."""
    return origin >= 1 and 0 <= sender <= origin - 2


def build_zigzag_token_ring(ranks, seq_len, heads, head_dim, route: str = "ring") -> Schedule:
    """Causal TokenRing over the zigzag partition (ref engine.py:306-366).

    ``route="ring"`` is the reference schedule, message for message.
    ``route="direct"`` (NOT a reference schedule) keeps
    every compute of the reference at the same rank and step but stops
    carrying a low sub-chunk through the hosts that do not compute it
    (ref engine.py:346-353 forwards it through hosts origin+1..P-1): origin
    o keeps its low chunk o until step P-o-1 and then sends it directly to
    host 0, which needs it at step P-o, over the NVSwitch full mesh.  It
    arrives in the same step and the same buffer position as on the ring,
    so no extra buffers exist; the Q bytes drop by (P-1)(P-2)/2 chunk-hops
    out of (P-1)(2P-1)."""
    if route not in ("ring", "direct"):
        raise ConfigError(f"route must be 'ring' or 'direct', got {route!r}")
    direct = route == "direct"
    kind = "zigzag-token-ring-direct" if direct else "zigzag-token-ring"
    part = split_zigzag(seq_len, ranks)
    if ranks == 1:
        return _trivial(kind, part, heads, head_dim, True)
    P = ranks
    c = seq_len // (2 * P)
    chunks = tuple(Chunk(a, a * c, (a + 1) * c, min(a, 2 * P - 1 - a)) for a in range(2 * P))
    oe = out_lse_elements(c, heads, head_dim)
    computed = {}          # (rank, step) -> q chunks computed
    steps, final = [], StepPlan.empty(P)
    for i in range(P):
        plan = StepPlan.empty(P)
        for r in range(P):
            o = (r - i) % P
            mine = (r, 2 * P - 1 - r)
            done = []
            for a in zigzag_alive(P, o, i):
                hit = False
                for b in mine:
                    if a > b:
                        plan.computes[r].append(ComputePlan(a, b, MaskSpec.none(), i == 0))
                        hit = True
                    elif a == b:
                        plan.computes[r].append(ComputePlan(
                            a, b, MaskSpec.causal(a * c, b * c), i == 0))
                        hit = True
                if hit:
                    done.append(a)
            computed[r, i] = tuple(done)
            if i < P - 1:
                carried = zigzag_alive(P, o, i + 1)
                if direct and o >= 1 and not _direct_carries_low(P, o, r):
                    carried = tuple(a for a in carried if a != o)
                if direct and r >= 1 and i == P - r - 1:
                    if (r + 1) % P == 0:       # host 0 is the ring successor: one message
                        carried = (r,) + tuple(a for a in carried if a != r)
                    else:
                        plan.sends[r].append(MsgPlan(r, 0, MsgKind.Q_BLOCK, (r,),
                                                     q_elements(c, heads, head_dim)))
                plan.sends[r].append(MsgPlan(r, (r + 1) % P, MsgKind.Q_BLOCK, carried,
                                             q_elements(len(carried) * c, heads, head_dim)))
            if i >= 2:
                ids = computed[r, i - 1]
                plan.sends[r].append(MsgPlan(r, (r - i + 1) % P, MsgKind.OUT_LSE, ids,
                                             len(ids) * oe))
        steps.append(plan)
    for r in range(P):
        ids = computed[r, P - 1]
        final.sends[r].append(MsgPlan(r, (r + 1) % P, MsgKind.OUT_LSE, ids, len(ids) * oe))
    return _wire_merges(Schedule(kind, P, heads, head_dim, True, part, chunks, steps, final))


def build_schedule(kind: str, ranks, seq_len, heads, head_dim, causal=None,
                   nodes: int = 1) -> Schedule:
    """Name-based front door: "ring" | "token-ring" | "zigzag-token-ring" |
    "hybrid" (``nodes`` must divide ``ranks``) | "zigzag-token-ring-direct"
    (non-reference Q routing, see ``build_zigzag_token_ring``)."""
    if kind == "hybrid":
        if causal:
            raise ConfigError("hybrid is non-causal; use zigzag-token-ring")
        if nodes < 1 or ranks % nodes:
            raise ConfigError(f"nodes must divide ranks (got ranks={ranks}, nodes={nodes})")
        return build_hybrid(nodes, ranks // nodes, seq_len, heads, head_dim)
    if kind == "ring":
        return build_ring_attention(ranks, seq_len, heads, head_dim, bool(causal))
    if kind == "token-ring":
        if causal:
            raise ConfigError("token-ring is non-causal; use zigzag-token-ring")
        return build_token_ring(ranks, seq_len, heads, head_dim)
    if kind == "zigzag-token-ring":
        if causal is False:
            raise ConfigError("zigzag-token-ring is causal")
        return build_zigzag_token_ring(ranks, seq_len, heads, head_dim)
    if kind == "zigzag-token-ring-direct":
        if causal is False:
            raise ConfigError("zigzag-token-ring-direct is causal")
        return build_zigzag_token_ring(ranks, seq_len, heads, head_dim, route="direct")
    raise ConfigError(f"unknown schedule kind {kind!r}")


# ----------------------------------------------------------------- traces
@dataclass(frozen=True)
class MsgRecord:
    step: int
    src: int
    dst: int
    kind: MsgKind
    elements: int


@dataclass(frozen=True)
class ComputeRecord:
    step: int
    rank: int
    flops: int


@dataclass
class MessageTrace:
    ranks: int
    n_steps: int
    messages: list = field(default_factory=list)
    computes: list = field(default_factory=list)


def trace_from_schedule(sched: Schedule) -> MessageTrace:
    """ref engine.py:399-417: the static message / flop trace."""
    tr = MessageTrace(sched.ranks, sched.n_steps)
    for step, plan in enumerate(sched.all_plans()):
        for r in range(sched.ranks):
            for cp in plan.computes[r]:
                tr.computes.append(ComputeRecord(step, r, compute_flops(
                    cp.mask, sched.chunks[cp.q_chunk].tokens, sched.chunks[cp.kv_chunk].tokens,
                    sched.heads, sched.head_dim)))
            for m in plan.sends[r]:
                tr.messages.append(MsgRecord(step, m.src, m.dst, m.kind, m.payload_elements))
    return tr


@dataclass
class VolumeReport:
    ranks: int
    n_steps: int
    entries: dict

    def elements(self, step, rank, kind) -> int:
        return self.entries.get((step, rank, kind), 0)

    def forward_elements(self, step=None, rank=None) -> int:
        return self._total(FORWARD_KINDS, step, rank)

    def reverse_elements(self, step=None, rank=None) -> int:
        return self._total((MsgKind.OUT_LSE,), step, rank)

    def _total(self, kinds, step, rank):
        return sum(n for (s, r, k), n in self.entries.items()
                   if k in kinds and (step is None or s == step) and (rank is None or r == rank))


def comm_volume(sched: Schedule) -> VolumeReport:
    ent = {}
    for step, plan in enumerate(sched.all_plans()):
        for r in range(sched.ranks):
            for m in plan.sends[r]:
                key = (step, r, m.kind)
                ent[key] = ent.get(key, 0) + m.payload_elements
    return VolumeReport(sched.ranks, sched.n_steps, ent)


def total_flops(sched: Schedule) -> int:
    return sum(c.flops for c in trace_from_schedule(sched).computes)


# ----------------------------------------------------------------- grouping
def _visible(sched, a, b):
    """(q chunk a, kv chunk b): 'none' | 'causal' | 'masked' by global position."""
    qa, kb = sched.chunks[a], sched.chunks[b]
    if not sched.causal or qa.start >= kb.stop - 1:
        return MaskKind.NONE
    if qa.stop - 1 < kb.start:
        return MaskKind.FULLY_MASKED
    return MaskKind.CAUSAL


def group_computes(sched: Schedule, computes) -> tuple | None:
    """Collapse one rank's computes of a step into (q ids, kv ids, accumulate)
    when they are exactly 'every q chunk x every kv chunk' under positional
    causality -- then one segmented launch reproduces them.  Returns None if
    the plan is not of that form."""
    if not computes:
        return (), (), None
    qs, ks = [], []
    for cp in computes:
        if cp.q_chunk not in qs:
            qs.append(cp.q_chunk)
        if cp.kv_chunk not in ks:
            ks.append(cp.kv_chunk)
    acc = {cp.accumulate for cp in computes}
    if len(acc) != 1 or len(qs) > 4 or len(ks) > 4:
        return None
    want = set()
    for a in qs:
        for b in ks:
            vis = _visible(sched, a, b)
            if vis is not MaskKind.FULLY_MASKED:
                want.add((a, b, vis))
    got = set()
    for cp in computes:
        if cp.mask.kind is MaskKind.FULLY_MASKED:
            continue
        if cp.mask.kind is MaskKind.CAUSAL:
            ca, cb = sched.chunks[cp.q_chunk], sched.chunks[cp.kv_chunk]
            if (cp.mask.q_offset, cp.mask.k_offset) != (ca.start, cb.start):
                return None
        got.add((cp.q_chunk, cp.kv_chunk, _visible(sched, cp.q_chunk, cp.kv_chunk)))
        if cp.mask.kind is MaskKind.NONE and _visible(sched, cp.q_chunk, cp.kv_chunk) is not MaskKind.NONE:
            return None
    if got != want:
        return None
    return tuple(qs), tuple(ks), acc.pop()


# ----------------------------------------------------------------- executor
def execute(sched: Schedule, q, k, v, causal: bool | None = None, timeline: list | None = None,
            check_finite: bool = True):
    """Run a schedule with all simulated ranks on the current GPU.

    Same contract as ``ringsim.engine.execute`` (ref engine.py:468-638):
    returns ({rank: Partial over the rank's home chunks in start order},
    MessageTrace) and raises ScheduleError naming step and rank when a
    compute touches a chunk that was never delivered or a return is
    unexpected.  Partials are float32 (out) / float32 (lse) on the device.
    If ``timeline`` is a list, (step, rank, start_event, end_event) CUDA
    event pairs bracketing every rank's attention launch are appended to it
    (the measured counterpart of the reference's netsim compute lane).
    ``check_finite=False`` skips the non-finite input check (ref core.py:96-104),
    a device-to-host read that blocks the host until the GPU is idle -- for
    timing loops that checked their inputs once beforehand.
    """
    if causal is not None and causal != sched.causal:
        raise ConfigError(f"schedule was built causal={sched.causal}, got causal={causal}")
    q, k, v = check_qkv(q, k, v, check_finite)
    shape = (sched.partition.seq_len, sched.heads, sched.head_dim)
    if tuple(q.shape) != shape:
        raise DimensionError(f"q must have shape {shape}, got {tuple(q.shape)}")
    if k.shape != q.shape or v.shape != q.shape:
        raise DimensionError("q, k, v must share one global shape")
    S, H, D = shape
    dev = q.device
    P = sched.ranks
    ch = sched.chunks
    q_res = {r: set() for r in range(P)}
    kv_res = {r: set() for r in range(P)}
    for c in ch:
        q_res[c.home].add(c.id)
        kv_res[c.home].add(c.id)
    acc_out = torch.empty(shape, dtype=torch.float32, device=dev)
    acc_lse = torch.empty((H, S), dtype=torch.float32, device=dev)
    fresh = {c.id for c in ch}      # chunks whose accumulator rows are still Partial.empty
    stage_out = [torch.empty(shape, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    stage_lse = [torch.empty((H, S), dtype=torch.float32, device=dev) for _ in range(2)]
    stash = {r: None for r in range(P)}       # rank -> (stage index, chunk ids)
    in_flight = []
    trace = MessageTrace(P, sched.n_steps)

    def merge_rows(cid, buf):
        c = ch[cid]
        if cid in fresh:           # first contribution: empty accumulator rows
            kernels.partial_init_(acc_out[c.start:c.stop], acc_lse[:, c.start:c.stop])
            fresh.discard(cid)
        kernels.merge_state_(acc_out[c.start:c.stop], acc_lse[:, c.start:c.stop],
                             stage_out[buf][c.start:c.stop], stage_lse[buf][:, c.start:c.stop])

    def fold(step, rank, msg):
        src, dst, kind, ids, payload = msg
        for cid in ids:
            if ch[cid].home != rank:
                raise ScheduleError(f"step {step} rank {rank}: returned chunk {cid} homes at "
                                    f"rank {ch[cid].home}")
            merge_rows(cid, payload)

    for step, plan in enumerate(sched.all_plans()):
        buf = step % 2
        arrivals = {r: [] for r in range(P)}
        for m in in_flight:
            arrivals[m[1]].append(m)
        in_flight = []
        for r in range(P):
            returned = []
            for m in arrivals[r]:
                if m[2] is MsgKind.Q_BLOCK:
                    q_res[r].update(m[3])
                elif m[2] is MsgKind.KV_BLOCK:
                    kv_res[r].update(m[3])
                else:
                    returned.append(m)
            expected = sorted((mp.src, tuple(mp.chunk_ids)) for mp in plan.merges[r])
            got = sorted((m[0], tuple(m[3])) for m in returned)
            if expected != got:
                raise ScheduleError(f"step {step} rank {r}: expected returns {expected}, got {got}")
            for mp in plan.merges[r]:
                m = next(x for x in returned if (x[0], tuple(x[3])) == (mp.src, tuple(mp.chunk_ids)))
                returned.remove(m)
                fold(step, r, m)
        outgoing = {}
        for r in range(P):
            for m in plan.sends[r]:
                if m.kind is MsgKind.OUT_LSE:
                    held = stash[r]
                    if held is None or set(held[1]) != set(m.chunk_ids):
                        raise ScheduleError(
                            f"step {step} rank {r}: OUT_LSE send expects chunks {m.chunk_ids}, "
                            f"stash holds {sorted(held[1]) if held else None}")
                    outgoing[r] = held[0]
                    stash[r] = None
        for r in range(P):
            cps = plan.computes[r]
            for cp in cps:
                if cp.q_chunk not in q_res[r]:
                    raise ScheduleError(f"step {step} rank {r}: q chunk {cp.q_chunk} not resident")
                if cp.kv_chunk not in kv_res[r]:
                    raise ScheduleError(f"step {step} rank {r}: kv chunk {cp.kv_chunk} not resident")
                trace.computes.append(ComputeRecord(step, r, compute_flops(
                    cp.mask, ch[cp.q_chunk].tokens, ch[cp.kv_chunk].tokens, H, D)))
            if not cps:
                continue
            g = group_computes(sched, cps)
            if g is None:
                raise ScheduleError(f"step {step} rank {r}: mixed accumulate flags or a compute "
                                    "set the segmented kernel cannot express")
            qs, ks, accumulate = g
            q_segs = [(ch[a].start, ch[a].tokens, ch[a].start) for a in qs]
            kv_segs = [(ch[b].start, ch[b].tokens, ch[b].start) for b in ks]
            if timeline is not None:
                ev0 = torch.cuda.Event(enable_timing=True)
                ev0.record()
            # accumulate-only rows that are the chunks' first contribution go
            # straight into the float32 accumulator (no init, no merge)
            direct = accumulate and all(a in fresh and ch[a].home == r for a in qs)
            kernels.attention_segments(q, k, v, q_segs, kv_segs, sched.causal,
                                       acc_out if direct else stage_out[buf],
                                       acc_lse if direct else stage_lse[buf])
            if timeline is not None:
                ev1 = torch.cuda.Event(enable_timing=True)
                ev1.record()
                timeline.append((step, r, ev0, ev1))
            if direct:
                fresh.difference_update(qs)
            elif accumulate:
                for a in sorted(qs):
                    if ch[a].home != r:
                        raise ScheduleError(f"step {step} rank {r}: accumulate for chunk {a} "
                                            f"homed at rank {ch[a].home}")
                    merge_rows(a, buf)
            else:
                stash[r] = (buf, tuple(qs))
        for r in range(P):
            for m in plan.sends[r]:
                if m.kind is MsgKind.Q_BLOCK:
                    for cid in m.chunk_ids:
                        if cid not in q_res[r]:
                            raise ScheduleError(f"step {step} rank {r}: cannot send q chunk "
                                                f"{cid}, not resident")
                        q_res[r].discard(cid)
                    in_flight.append((r, m.dst, m.kind, tuple(m.chunk_ids), None))
                elif m.kind is MsgKind.KV_BLOCK:
                    (cid,) = m.chunk_ids
                    if cid not in kv_res[r]:
                        raise ScheduleError(f"step {step} rank {r}: cannot send kv chunk "
                                            f"{cid}, not resident")
                    kv_res[r].discard(cid)
                    in_flight.append((r, m.dst, m.kind, (cid,), None))
                else:
                    in_flight.append((r, m.dst, m.kind, tuple(m.chunk_ids), outgoing[r]))
                trace.messages.append(MsgRecord(step, r, m.dst, m.kind, m.payload_elements))
    for cid in sorted(fresh):      # rows nobody contributed to stay Partial.empty
        c = ch[cid]
        kernels.partial_init_(acc_out[c.start:c.stop], acc_lse[:, c.start:c.stop])
    fresh.clear()
    last = sched.n_steps - 1
    for m in in_flight:
        if m[2] is not MsgKind.OUT_LSE:
            raise ScheduleError(f"step {last} rank {m[0]}: {m[2].value} message left in flight "
                                "after the final step")
        fold(last, m[1], m)
    del stage_out, stage_lse           # release the step buffers before the output copies
    outputs = {}
    for r in range(P):
        rng = sched.partition.ranges(r)
        outputs[r] = Partial(torch.cat([acc_out[a:b] for a, b in rng], 0),
                             torch.cat([acc_lse[:, a:b] for a, b in rng], 1))
    return outputs, trace
