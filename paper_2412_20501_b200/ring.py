"""Multi-GPU TokenRing: one process per GPU, torch.distributed for the
plumbing (NCCL P2P over NVLink/NVSwitch), sm_100a kernels for the math.

Per rank r and step i (schedule from ``engine.build_zigzag_token_ring`` /
``build_token_ring``; semantics of ref engine.py:233-366, 468-638):

    wait(comm[i-1])            Q_i has arrived; OUT returned at i-1 has arrived
    merge returned OUT         lse-merge kernel into the float32 accumulator
    issue comm[i]              send Q_i -> r+1, recv Q_{i+1} <- r-1,
                               send OUT(step i-1) -> home, recv OUT <- sender
    compute[i]                 ONE segmented attention launch (all q sub-chunks
                               of the traveling set x both local kv sub-chunks)

so the forward Q stream and the reverse OUT stream of step i run on the NCCL
stream concurrently with compute[i] on the compute stream.  The final phase
returns the last step's rows.  Double-buffered traveling-Q and output
buffers make every hazard an ordering on the compute stream.

Outputs stay sharded: rank r returns its home chunks in start order, exactly
what ref ``engine.execute`` returns per rank, so ``global_reorder`` works.
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import kernels
from .core import MaskKind, Partial
from .engine import (MsgKind, build_hybrid, build_ring_attention, build_token_ring,
                     build_zigzag_token_ring, group_computes)
from .errors import ConfigError, DimensionError, ScheduleError


# nccl:  torch.distributed batch_isend_irecv on NCCL's streams
# ipc:   copy engines into CUDA-IPC-mapped peer buffers + device sequence flags
# fused: ipc for Q; the OUT_LSE messages are written by the attention kernel's
#        epilogue straight into the home rank's receive slot (NVLink stores)
TRANSPORTS = ("nccl", "ipc", "fused")
# token-ring: TokenRing (zigzag when causal, contiguous otherwise; hybrid with
#             nodes > 1) -- Q forward, OUT_LSE reverse
# ring:       Ring Attention, KV forward only (the reference's baseline)
SCHEDULES = ("token-ring", "ring")


class CudaOps:
    """Device ops of the product path (libtokenring.so)."""

    def __init__(self, device):
        self.device = torch.device(device)

    def attention(self, q, k, v, q_segs, kv_segs, causal, out, lse):
        kernels.attention_segments(q, k, v, q_segs, kv_segs, causal, out, lse)

    def merge_(self, acc_out, acc_lse, blk_out, blk_lse):
        kernels.merge_state_(acc_out, acc_lse, blk_out, blk_lse)

    def merge_n_(self, acc_out, acc_lse, blocks):
        kernels.merge_n_(acc_out, acc_lse, blocks)

    def init_(self, acc_out, acc_lse):
        kernels.partial_init_(acc_out, acc_lse)

    def event(self):
        return torch.cuda.Event(enable_timing=True)

    def record(self, ev):
        ev.record()


@dataclass
class RankStep:
    step: int
    q_layout: tuple          # chunk ids of the traveling Q buffer, in row order
    q_ids: tuple             # q chunks computed this step
    kv_ids: tuple            # local kv chunks used
    accumulate: bool | None
    send_q: list             # [(dst, ids, from_home)]  from_home: rows of the local shard
    recv_q: list             # [(src, ids)]  union (start order) = next step's buffer layout
    send_out: tuple | None   # (dst, ids)   rows from the previous step's output
    recv_out: list           # [(src, ids)]  to merge after this step's comm
    # KV residency (hybrid schedules rotate KV across nodes, ref engine.py:233-290):
    kv_layout: tuple = ()    # kv chunk ids of the store this step reads, in row order
    kv_store: int = -1       # -1: the local shard; k >= 0: the k-th received KV block
    send_kv: tuple | None = None   # (dst, ids) of the store, sent after this step
    recv_kv: tuple | None = None   # (src, ids) received during this step
    q_slot: int = -1         # traveling-Q buffer holding q_layout (-1: the local shard)


def compile_rank(sched, rank: int) -> list:
    """This rank's step program, derived from the schedule's plans."""
    P = sched.ranks
    plans = sched.all_plans()
    home = tuple(c.id for c in sorted((c for c in sched.chunks if c.home == rank),
                                      key=lambda c: c.start))
    layout, q_slot = home, -1
    kv_layout, kv_store, n_kv_recv = home, -1, 0
    start = {c.id: c.start for c in sched.chunks}
    prog = []
    for i, plan in enumerate(plans):
        g = group_computes(sched, plan.computes[rank])
        if g is None:
            raise ScheduleError(f"step {i} rank {rank}: compute set not expressible as one launch")
        q_ids, kv_ids, acc = g
        if all(cp.mask.kind is MaskKind.FULLY_MASKED for cp in plan.computes[rank]):
            # the causal ring's blocks above the diagonal (ref engine.py:216-223):
            # identity partials, nothing to launch or merge
            q_ids, kv_ids, acc = (), (), None
        send_q, recv_q, send_out, send_kv, recv_kv = [], [], None, None, None
        for m in plan.sends[rank]:
            if m.kind is MsgKind.Q_BLOCK:
                ids = tuple(m.chunk_ids)
                if all(a in layout for a in ids):
                    send_q.append((m.dst, ids, i == 0))
                elif all(a in home for a in ids):
                    send_q.append((m.dst, ids, True))      # kept at its origin (direct route)
                else:
                    raise ScheduleError(f"step {i} rank {rank}: cannot send q chunks {ids}")
            elif m.kind is MsgKind.OUT_LSE:
                send_out = (m.dst, tuple(m.chunk_ids))
            else:
                ids = tuple(m.chunk_ids)
                if send_kv is not None or not all(b in kv_layout for b in ids):
                    raise ScheduleError(f"step {i} rank {rank}: cannot send kv chunks {ids}")
                send_kv = (m.dst, ids)
        recv_out = []
        for src in range(P):
            for m in plan.sends[src]:
                if m.dst != rank:
                    continue
                if m.kind is MsgKind.Q_BLOCK:
                    recv_q.append((src, tuple(m.chunk_ids)))
                elif m.kind is MsgKind.OUT_LSE:
                    recv_out.append((src, tuple(m.chunk_ids)))
                else:
                    if recv_kv is not None:
                        raise ScheduleError(f"step {i} rank {rank}: two kv blocks in one step")
                    recv_kv = (src, tuple(m.chunk_ids))
        for a in q_ids:
            if a not in layout:
                raise ScheduleError(f"step {i} rank {rank}: q chunk {a} not resident")
        for b in kv_ids:
            if b not in kv_layout:
                raise ScheduleError(f"step {i} rank {rank}: kv chunk {b} not resident")
        prog.append(RankStep(i, layout, q_ids, kv_ids, acc, send_q, recv_q, send_out, recv_out,
                             kv_layout, kv_store, send_kv, recv_kv, q_slot))
        if recv_q:
            # Q received at step i lands in traveling buffer (i+1) % 2
            layout = tuple(sorted((a for _, ids in recv_q for a in ids), key=start.get))
            q_slot = (i + 1) % 2
        if recv_kv is not None:
            if send_kv is None:
                raise ScheduleError(f"step {i} rank {rank}: kv received without handing one on")
            kv_layout, kv_store, n_kv_recv = recv_kv[1], n_kv_recv, n_kv_recv + 1
    return prog


def _nvtx_push(name):
    # NVTX ranges per TokenRing step (host side; visible in nsys / ncu --nvtx)
    torch.cuda.nvtx.range_push(name)


def _nvtx_pop():
    torch.cuda.nvtx.range_pop()


def _ptrs(*ts):
    return tuple(t.data_ptr() for t in ts)


def _rows(layout, ids, c):
    """Contiguous row range of ``ids`` inside a buffer laid out as ``layout``."""
    idx = [layout.index(a) for a in ids]
    if idx != list(range(idx[0], idx[0] + len(idx))):
        raise ScheduleError(f"chunks {ids} are not contiguous in buffer {layout}")
    return idx[0] * c, (idx[0] + len(idx)) * c


@dataclass
class FusedPlan:
    """Message bookkeeping of the ``fused`` transport for one rank.

    push[s] = (msg, dst, row0, row1): computing step s writes its rows
        [row0, row1) of the traveling-Q layout (all of them, in layout order)
        straight into ``dst``'s receive slot for message msg -- the OUT_LSE
        message the reference sends at step msg = s + 1 (engine.py:346-353).
    recv[k] = (src, ids, slot): message k arrives in my slot ``slot`` (one
        slot per message, in step order, never reused within a forward);
        all of them are folded into the accumulator by ONE n-way merge per
        home chunk after the last step -- the MergePlans of engine.py:187-200
        and 620-628 applied at once (the merge is associative).
    """
    push: dict
    recv: dict

    def slot_of(self, k):
        return self.recv[k][2]

    def merge_groups(self, home_ids):
        """For each home chunk: [(slot, position of the chunk in the message)]."""
        return {a: [(slot, ids.index(a)) for _, (_, ids, slot) in sorted(self.recv.items())
                    if a in ids] for a in home_ids}


def fused_plan(prog, c) -> FusedPlan:
    """Derive the push / receive program of one rank from its step program
    (``compile_rank``); ScheduleError if a message is not a whole step's
    rows (never the case for the reference's token-ring schedules)."""
    push, recv = {}, {}
    for k, st in enumerate(prog):
        if st.send_out is not None:
            dst, ids = st.send_out
            prev = prog[k - 1]
            if prev.accumulate or sorted(prev.q_ids) != sorted(ids):
                raise ScheduleError(f"step {k}: OUT message {ids} is not step {k - 1}'s rows "
                                    f"{prev.q_ids}; the fused transport cannot push it")
            a, b = _rows(prev.q_layout, ids, c)
            push[k - 1] = (k, dst, a, b)
        if st.recv_out:
            if len(st.recv_out) != 1:
                raise ScheduleError(f"step {k}: more than one return per step")
            src, ids = st.recv_out[0]
            recv[k] = (src, tuple(ids), len(recv))
    return FusedPlan(push, recv)


class TokenRingAttention:
    """TokenRing forward on this process's rank of ``group``.

    ``q_loc/k_loc/v_loc``: this rank's (S/P, H, D) bf16 shard -- its partition
    ranges concatenated in start order (``partition.gather_local``).
    Returns a float32 Partial over the same rows.

    ``overlap_steps`` (ipc / fused): each step's message waits and attention
    launch are programmatic dependent launches of the previous step, so its
    CTAs start on the SMs the previous step's last wave frees; results are
    bit-identical to plain stream-ordered steps (``overlap_steps=False``).
    """

    def __init__(self, seq_len, heads, head_dim, causal=True, group=None, ops=None,
                 device=None, record_timeline=False, transport="nccl", route="ring", nodes=1,
                 schedule="token-ring", overlap_steps=True):
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if schedule not in SCHEDULES:
            raise ConfigError(f"schedule must be one of {SCHEDULES}, got {schedule!r}")
        if route != "ring" and not causal:
            raise ConfigError("route='direct' applies to the causal zigzag schedule only")
        if schedule == "ring":
            # Ring Attention, the config-4 baseline (ref engine.py:203-230):
            # contiguous shards, every rank keeps its Q and accumulates locally,
            # KV blocks rotate to rank+1 -- carried by the same KV-store
            # machinery as the hybrid schedule's node hand-offs
            if route != "ring" or nodes > 1:
                raise ConfigError("schedule='ring' takes no route or nodes")
            self.sched = build_ring_attention(self.P, seq_len, heads, head_dim, causal)
        elif nodes > 1:
            # the reference's multi-node schedule (ref engine.py:298-303): TokenRing
            # inside each group of P/nodes ranks, KV rotated across the groups
            if causal:
                raise ConfigError("hybrid schedule requires causal=False (ref engine.py:298-303)")
            if self.P % nodes:
                raise ConfigError(f"world size {self.P} is not a multiple of nodes={nodes}")
            self.sched = build_hybrid(nodes, self.P // nodes, seq_len, heads, head_dim)
        elif causal:
            self.sched = build_zigzag_token_ring(self.P, seq_len, heads, head_dim, route=route)
        else:
            self.sched = build_token_ring(self.P, seq_len, heads, head_dim)
        self.causal = causal
        self.S, self.H, self.D = seq_len, heads, head_dim
        self.part = self.sched.partition
        self.local_rows = self.part.owned_tokens(self.rank)
        self.c = self.sched.chunks[0].tokens
        self.prog = compile_rank(self.sched, self.rank)
        self.has_kv = any(st.recv_kv is not None for st in self.prog)
        self._progs = {self.rank: self.prog}
        self._layouts = {}
        # Step 0 computes every home chunk with accumulate=True (TokenRing and
        # zigzag TokenRing alike): those rows are the accumulator's first
        # contribution, so the kernel writes them into it as float32 -- no
        # Partial.empty fill, no bf16 block, no merge pass.
        st0 = self.prog[0]
        self.direct_first = bool(st0.accumulate) and sorted(st0.q_ids) == sorted(st0.q_layout)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.ops = ops if ops is not None else CudaOps(device)
        self.device = self.ops.device
        self.record_timeline = record_timeline
        # ipc / fused: each step's message waits and attention launch are
        # programmatic dependent launches, so a step's grid starts on the SMs
        # the previous step's last wave frees (one rank's P=8 step chain: +17 %
        # at 32K, +3 % at 128K, scripts/probe_pdl.py); a step reads only
        # messages its own flag waits covered, never the previous grid's output
        self.overlap_steps = bool(overlap_steps)
        self.timeline = []
        self._graph = None              # (CUDAGraph, input pointers) after capture()
        if transport not in TRANSPORTS:
            raise ConfigError(f"transport must be one of {TRANSPORTS}, got {transport!r}")
        self.transport = transport if self.P > 1 else "nccl"
        self.fplan = self.fplans = None
        if self.transport == "fused":
            # every rank's plan: a sender needs the slot index its message
            # has at the home
            self.fplans = {r: fused_plan(compile_rank(self.sched, r) if r != self.rank
                                         else self.prog, self.c) for r in range(self.P)}
            self.fplan = self.fplans[self.rank]
        self._alloc()
        if self.transport in ("ipc", "fused"):
            self._ipc_setup()

    def _alloc(self):
        rows, H, D, dev = self.local_rows, self.H, self.D, self.device
        bf = torch.bfloat16
        self.qbuf = [torch.empty((rows, H, D), dtype=bf, device=dev) for _ in range(2)]
        self.obuf = [torch.empty((rows, H, D), dtype=bf, device=dev) for _ in range(2)]
        self.lbuf = [torch.empty((H, rows), dtype=torch.float32, device=dev) for _ in range(2)]
        self.lse_send = torch.empty((H, rows), dtype=torch.float32, device=dev)
        recv_rows = rows if self.transport != "fused" else 1     # fused: per-message slots
        self.out_recv = torch.empty((recv_rows, H, D), dtype=bf, device=dev)
        self.lse_recv = torch.empty((H, recv_rows), dtype=torch.float32, device=dev)
        self.acc_out = torch.empty((rows, H, D), dtype=torch.float32, device=dev)
        self.acc_lse = torch.empty((H, rows), dtype=torch.float32, device=dev)
        self.slots = []
        # received KV blocks (hybrid schedules): two stores, the k-th receive
        # lands in kvbuf[k % 2]
        self.kvbuf = ([(torch.empty((rows, H, D), dtype=bf, device=dev),
                        torch.empty((rows, H, D), dtype=bf, device=dev)) for _ in range(2)]
                      if self.has_kv else [])
        if self.transport == "fused":
            # one receive slot per message of a forward (bf16 rows + lse), all
            # folded by one n-way merge at the end; and the launch counter the
            # pushing kernels use for their done flag
            for k, (_, ids, _) in sorted(self.fplan.recv.items()):
                n = len(ids) * self.c
                self.slots.append((torch.empty((n, H, D), dtype=bf, device=dev),
                                   torch.empty((H, n), dtype=torch.float32, device=dev)))
            # (one per step: overlapping step launches count separately)
            self.done_count = torch.zeros(len(self.prog), dtype=torch.int32, device=dev)

    # -- transport -----------------------------------------------------------
    def _comm(self, sends, recvs):
        if self.P == 1 or not (sends or recvs):
            return []
        backend = dist.get_backend(self.group)
        if backend == "nccl":
            ops = [dist.P2POp(dist.isend, t, self._global(p), self.group) for p, t in sends]
            ops += [dist.P2POp(dist.irecv, t, self._global(p), self.group) for p, t in recvs]
            return dist.batch_isend_irecv(ops)
        reqs = [dist.isend(t, self._global(p), self.group) for p, t in sends]
        reqs += [dist.irecv(t, self._global(p), self.group) for p, t in recvs]
        return reqs

    def _global(self, r):
        return r if self.group is None else dist.get_global_rank(self.group, r)

    # -- one forward -----------------------------------------------------------
    # -- copy-engine transport (CUDA IPC / NVLink peer memory) ----------------
    # Every rank exposes its receive buffers and a flag block to all peers
    # (torch's CUDA IPC handles, exchanged once over the process group).  A
    # send is a cudaMemcpyAsync straight into the peer's buffer on this rank's
    # copy stream -- copy engines, no SMs taken from the attention kernel --
    # followed by a release store to the peer's sequence flag.
    # Values are call-relative: call n uses base_n = BASE0 + n*L (L = steps of
    # the rank program) and every flag
    # only grows, so consecutive calls need no reset, no device sync and no
    # barrier -- each flag's value at the end of call n is exactly its initial
    # condition for call n+1 (set once for call 0 in _ipc_setup).
    #   flags[0] fin     : base of the last call whose received messages I have
    #                      folded (fused: a sender may reuse my slots)
    #   flags[1] q_free  : highest step whose traveling-Q slot I am done with
    #   flags[2] o_ready : highest step whose returned OUT for me has landed
    #   flags[3] o_free  : step of the last returned OUT I have merged (base+1:
    #                      none yet this call, and the previous call's are)
    #   flags[4+s] q_ready from s: highest step whose Q from rank s has landed
    #              (one per source: the direct route has two Q senders per step)
    # fused transport (OUT pushed by the attention epilogue) adds
    #   flags[4+P+s]   o_ready of receive slot s (raised by the pushing kernel's
    #                  last CTA); slot s's buffers are shared as entries 5+2s, 6+2s
    def _ipc_setup(self):
        from torch.multiprocessing.reductions import reduce_tensor
        # ... flags[KVF] kv_ready: highest step whose KV block for me has landed
        self.KVF = 4 + self.P + len(self.prog) + 1
        self.flags = torch.zeros(self.KVF + 1, dtype=torch.int64, device=self.device)
        shared = [self.qbuf[0], self.qbuf[1], self.out_recv, self.lse_recv, self.flags]
        for o, l in self.slots:
            shared += [o, l]
        for kb, vb in self.kvbuf:          # entries after the slots (see _peer_kv)
            shared += [kb, vb]
        mine = [reduce_tensor(t) for t in shared]
        everyone = [None] * self.P
        dist.all_gather_object(everyone, mine, group=self.group)
        self.peer = {}
        for r in range(self.P):
            if r == self.rank:
                continue
            fn_args = everyone[r]
            self.peer[r] = [fn(*args) for fn, args in fn_args]
            # torch maps a peer's handles in the PEER device's context; our flag
            # and push kernels run on this device and dereference them directly
            peer_dev = self.peer[r][0].device.index
            if peer_dev != self.device.index:
                with torch.cuda.device(self.device):
                    kernels.enable_peer_access(peer_dev)
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.calls = 0
        # initial conditions of call 0, visible to every peer before anyone sends
        b = self._base(0)
        self.epoch = torch.full((1,), b, dtype=torch.int64, device=self.device)
        init = torch.full_like(self.flags, b - 1)
        init[0] = b - len(self.prog)    # "the call before 0" has been folded
        init[1] = b                     # step 0 runs on q_loc: slot 0 is free
        init[3] = b + 1                 # ipc: my single OUT receive buffer is free
        self.flags.copy_(init)
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)

    def _base(self, call):
        # call n's flag values live in [base_n - 1, base_n + L + 1], L = steps per call
        L = len(self.prog)
        return 2 * L + 8 + call * L

    def close(self):
        """Drop the peers' IPC-mapped buffers (call on every rank, then
        barrier, before the processes exit: a CUDA IPC producer must outlive
        its consumers' mappings)."""
        torch.cuda.synchronize(self.device)
        self.peer = {}
        kernels.poll_error()

    def progs(self, r):
        """Rank r's step program (compiled on demand; peers' slot indices)."""
        if r not in self._progs:
            self._progs[r] = compile_rank(self.sched, r)
        return self._progs[r]

    def _kv_store(self, st, k_loc, v_loc):
        """(k, v, layout, local) of the KV store step ``st`` reads."""
        if st.kv_store < 0:
            return k_loc, v_loc, st.kv_layout, True
        kb, vb = self.kvbuf[st.kv_store % 2]
        return kb, vb, st.kv_layout, False

    def _kv_segs(self, st, local):
        c = self.c
        if local:
            return [(self.part.local_offset(self.rank, self.sched.chunks[b].start), c,
                     self.sched.chunks[b].start) for b in st.kv_ids]
        return [(st.kv_layout.index(b) * c, c, self.sched.chunks[b].start) for b in st.kv_ids]

    def _peer_kv(self, r, slot):
        """Peer r's received-KV store ``slot`` (IPC-mapped)."""
        nslots = len(self.fplans[r].recv) if self.fplans else 0
        i0 = 5 + 2 * nslots + 2 * slot
        return self.peer[r][i0], self.peer[r][i0 + 1]

    def _flags_of(self, r):
        return self.flags if r == self.rank else self.peer[r][4]

    def _recv_slot(self, slot, r=None):
        """(out, lse) of fused receive slot ``slot`` -- mine, or peer r's."""
        if r is None or r == self.rank:
            return self.slots[slot]
        return self.peer[r][5 + 2 * slot], self.peer[r][6 + 2 * slot]

    @contextlib.contextmanager
    def _timed_copy(self, ev, key, stream, nbytes):
        """Timeline events around a copy-engine transfer on ``stream``."""
        if not self.record_timeline:
            yield
            return
        e0, e1 = self.ops.event(), self.ops.event()
        e0.record(stream)
        yield
        e1.record(stream)
        ev.setdefault(key, []).append((e0, e1, nbytes))

    def _forward_ipc(self, q_loc, k_loc, v_loc) -> Partial:
        c, rank, P, H = self.c, self.rank, self.P, self.H
        fused, fp = self.transport == "fused", self.fplan
        O0 = 4 + P                     # fused: o_ready flag of each receive slot
        # every flag value of this call is epoch + offset: the epoch (a device
        # int64, = base of call n) is read on the device and advanced at the
        # end, so the same enqueued sequence -- or a CUDA graph of it -- is
        # valid for every call
        E = self.epoch
        self.calls += 1
        cur = torch.cuda.current_stream(self.device)
        cs = self.copy_stream
        if not self.direct_first:
            self.ops.init_(self.acc_out, self.acc_lse)
        local_layout = self.prog[0].q_layout
        ev_comp, ev_out_sent = {}, {}
        self.timeline = []
        for st in self.prog:
            i = st.step
            ev = {}
            _nvtx_push(f"tokenring step {i}")
            if self.record_timeline:
                ev["start"] = self.ops.event()
                self.ops.record(ev["start"])
            # step i >= 1 after step i-1; every step releases the next one
            overlap = kernels.overlap_launches(after_prev=self.overlap_steps and i >= 1,
                                               release_next=self.overlap_steps)
            with overlap:
                if i >= 1 and (st.q_ids or st.send_q):
                    for src, _ in self.prog[i - 1].recv_q:              # Q_i has landed
                        kernels.flag_wait_(self.flags[4 + src:5 + src], i, cur, epoch=E)
                if i >= 1 and self.prog[i - 1].recv_out and not fused:
                    kernels.flag_wait_(self.flags[2:3], i - 1, cur, epoch=E)
                if i >= 1 and self.prog[i - 1].recv_kv is not None:    # KV for this phase
                    kernels.flag_wait_(self.flags[self.KVF:self.KVF + 1], i, cur, epoch=E)
            if self.record_timeline:
                ev["comm_ready"] = self.ops.event()
                self.ops.record(ev["comm_ready"])
            if i >= 1 and self.prog[i - 1].recv_out and not fused:
                # OUT sent to me at step i-1 has landed: merge it, free the buffer
                src, ids = self.prog[i - 1].recv_out[0]
                n = len(ids) * c
                self._merge_returned((ids, self.out_recv[:n],
                                      self.lse_recv.view(-1)[: H * n].view(H, n)), local_layout)
                kernels.flag_set_(self.flags[3:4], i - 1, cur, epoch=E)
            cur_q = self.qbuf[st.q_slot] if st.q_slot >= 0 else q_loc
            kst, vst, kv_lay, kv_local = self._kv_store(st, k_loc, v_loc)
            ev_q = torch.cuda.Event()
            ev_q.record(cur)
            if st.send_q or st.send_kv is not None:
                cs.wait_event(ev_q)
            if st.send_kv is not None:
                # hand this phase's KV to the next node's rank (ref engine.py:287-290),
                # into its receive store once it has finished the previous step
                dst, ids = st.send_kv
                a, b = _rows(kv_lay, ids, c)
                slot = sum(1 for t in self.progs(dst)[:i] if t.recv_kv is not None) % 2
                pk, pv = self._peer_kv(dst, slot)
                kernels.flag_wait_(self.peer[dst][4][1:2], i - 1, cs, epoch=E)
                with self._timed_copy(ev, "kv_copies", cs, 2 * (b - a) * H * self.D * 2):
                    kernels.copy_(pk[: b - a], kst[a:b], cs)
                    kernels.copy_(pv[: b - a], vst[a:b], cs)
                kernels.flag_set_(self.peer[dst][4][self.KVF:self.KVF + 1], i + 1, cs, epoch=E)
            for dst, ids, from_home in st.send_q:
                src_buf, src_layout = (q_loc, local_layout) if from_home else (cur_q, st.q_layout)
                a, b = _rows(src_layout, ids, c)
                d0, d1 = _rows(self._next_layout(dst, i), ids, c)
                kernels.flag_wait_(self.peer[dst][4][1:2], i - 1, cs, epoch=E)   # peer slot free
                with self._timed_copy(ev, "q_copies", cs, (b - a) * H * self.D * 2):
                    kernels.copy_(self.peer[dst][(i + 1) % 2][d0:d1], src_buf[a:b], cs)
                kernels.flag_set_(self.peer[dst][4][4 + rank:5 + rank], i + 1, cs, epoch=E)
            if st.send_out is not None and not fused:   # fused: pushed by step i-1's kernel
                dst, ids = st.send_out
                a, b = _rows(self.prog[i - 1].q_layout, ids, c)
                cs.wait_event(ev_comp[i - 1])
                # the home's single receive buffer is free once it has merged the
                # previous message it received (messages need not come every step:
                # the hybrid schedule skips the accumulate steps)
                prev = [t.step for t in self.progs(dst)[:i] if t.recv_out]
                kernels.flag_wait_(self.peer[dst][4][3:4], prev[-1] if prev else 1, cs, epoch=E)
                ob, lb = self.obuf[(i - 1) % 2], self.lbuf[(i - 1) % 2]
                ls = self.lse_send.view(-1)[: self.H * (b - a)].view(self.H, b - a)
                with torch.cuda.stream(cs):
                    ls.copy_(lb[:, a:b])
                with self._timed_copy(ev, "o_copies", cs, (b - a) * H * (2 * self.D + 4)):
                    kernels.copy_(self.peer[dst][2][: b - a], ob[a:b], cs)
                    kernels.copy_(self.peer[dst][3].view(-1)[: self.H * (b - a)], ls, cs)
                kernels.flag_set_(self.peer[dst][4][2:3], i, cs, epoch=E)
                ev_out_sent[i] = torch.cuda.Event()
                ev_out_sent[i].record(cs)
            if st.q_ids:
                if (i - 1) in ev_out_sent:                 # obuf[i%2] was read by that send
                    cur.wait_event(ev_out_sent[i - 1])
                q_segs = [(_rows(st.q_layout, (a,), c)[0], c, self.sched.chunks[a].start)
                          for a in st.q_ids]
                kv_segs = self._kv_segs(st, kv_local)
                buf = i % 2
                if self.record_timeline:
                    ev["attn_start"] = self.ops.event()
                    self.ops.record(ev["attn_start"])
                if i == 0 and self.direct_first:
                    with overlap:
                        self.ops.attention(cur_q, kst, vst, q_segs, kv_segs, self.causal,
                                           self.acc_out, self.acc_lse)
                elif fused and i in fp.push:
                    # compute + send in one kernel: rows go straight into the
                    # home's receive slot over NVLink; its last CTA raises the
                    # home's o_ready flag
                    # (the slot holds only message k, and the previous call's
                    # merge of it finished before this call's barrier)
                    k, dst, a, b = fp.push[i]
                    slot = self.fplans[dst].slot_of(k)
                    ob, lb = self._recv_slot(slot, dst)
                    ev["o_push_bytes"] = (b - a) * H * (2 * self.D + 4)   # carried by this launch
                    o = O0 + slot
                    with overlap:
                        # the home has folded the previous call's messages out of its slots
                        kernels.flag_wait_(self._flags_of(dst)[0:1], -len(self.prog), cur,
                                           epoch=E)
                        kernels.attention_segments_push(
                            cur_q, kst, vst, q_segs, kv_segs, self.causal, ob, lb, a,
                            self.done_count[i:i + 1], self._flags_of(dst)[o:o + 1], k, epoch=E)
                else:
                    with overlap:
                        self.ops.attention(cur_q, kst, vst, q_segs, kv_segs, self.causal,
                                           self.obuf[buf], self.lbuf[buf])
                if self.record_timeline:
                    ev["attn_end"] = self.ops.event()
                    self.ops.record(ev["attn_end"])
                    ev["attn_flops"] = self.step_flops(st)
                if st.accumulate and not (i == 0 and self.direct_first):
                    for a in st.q_ids:
                        r0, r1 = _rows(st.q_layout, (a,), c)
                        l0 = self.part.local_offset(rank, self.sched.chunks[a].start)
                        self.ops.merge_(self.acc_out[l0:l0 + c], self.acc_lse[:, l0:l0 + c],
                                        self.obuf[buf][r0:r1], self.lbuf[buf][:, r0:r1])
            ev_comp[i] = torch.cuda.Event()
            ev_comp[i].record(cur)
            if self.record_timeline:
                ev["computed"] = self.ops.event()
                self.ops.record(ev["computed"])
                self.timeline.append(ev)
            # step i is done here: my traveling-Q slot i%2 (and, in hybrid
            # schedules, the KV store read before this step) is free once
            # this step's compute and my own forward copies are done
            cs.wait_event(ev_comp[i])
            kernels.flag_set_(self.flags[1:2], i, cs, epoch=E)
            _nvtx_pop()
        last = self.prog[-1]
        if fused:
            self._merge_all_fused(cur, local_layout)
        elif last.recv_out:
            kernels.flag_wait_(self.flags[2:3], last.step, cur, epoch=E)
            src, ids = last.recv_out[0]
            n = len(ids) * c
            self._merge_returned((ids, self.out_recv[:n],
                                  self.lse_recv.view(-1)[: H * n].view(H, n)), local_layout)
        # hand the next call its initial conditions (next base = base + P):
        # everything received is folded, the OUT buffer is free, and both
        # traveling-Q slots are free once this call's computes are done
        L = len(self.prog)
        kernels.flag_set_(self.flags[0:1], 0, cur, epoch=E)
        kernels.flag_set_(self.flags[3:4], L + 1, cur, epoch=E)
        cs.wait_stream(cur)
        kernels.flag_set_(self.flags[1:2], L, cs, epoch=E)
        cur.wait_stream(cs)
        kernels.epoch_add_(E, L, cur)        # last: the next call's base
        return Partial(self.acc_out, self.acc_lse)

    def _merge_all_fused(self, cur, local_layout):
        """Wait for every pushed message, then fold all of them into the
        accumulator: one n-way merge per home chunk (tr_merge_n)."""
        fp, c, P = self.fplan, self.c, self.P
        ev = {}
        if self.record_timeline:
            ev["start"] = self.ops.event()
            self.ops.record(ev["start"])
        for k, (_, _, slot) in sorted(fp.recv.items()):
            kernels.flag_wait_(self.flags[4 + P + slot:5 + P + slot], k, cur, epoch=self.epoch)
        if self.record_timeline:
            ev["comm_ready"] = self.ops.event()
            self.ops.record(ev["comm_ready"])
            self.timeline.append(ev)
        for a, parts in fp.merge_groups(local_layout).items():
            if self.sched.chunks[a].home != self.rank:
                raise ScheduleError(f"rank {self.rank}: chunk {a} homes elsewhere")
            l0 = self.part.local_offset(self.rank, self.sched.chunks[a].start)
            blocks = [(self.slots[slot][0][j * c:(j + 1) * c],
                       self.slots[slot][1][:, j * c:(j + 1) * c]) for slot, j in parts]
            if blocks:
                self.ops.merge_n_(self.acc_out[l0:l0 + c], self.acc_lse[:, l0:l0 + c], blocks)

    def __call__(self, q_loc, k_loc, v_loc) -> Partial:
        """One forward over this rank's shard; returns this rank's home rows.

        The returned Partial's tensors are the runner's own float32
        accumulator (no copy is made): they hold this call's result only
        until the next call on the same runner, which overwrites them
        asynchronously on the device.  Clone them (or copy them out, as
        bench.py's e2e path does) before calling again.

        ipc / fused transports: a message that never arrives makes the
        device-side wait time out (30 s) instead of hanging or trapping;
        the next call (or ``close``) raises ScheduleError for it."""
        if self._graph is not None and self._graph[1] == _ptrs(q_loc, k_loc, v_loc):
            if self.transport in ("ipc", "fused"):
                kernels.poll_error()
            self._graph[0].replay()
            return Partial(self.acc_out, self.acc_lse)
        return self._forward(q_loc, k_loc, v_loc)

    def _forward(self, q_loc, k_loc, v_loc) -> Partial:
        if self.transport in ("ipc", "fused"):
            kernels.poll_error()
            shape = (self.local_rows, self.H, self.D)
            for n, t in (("q", q_loc), ("k", k_loc), ("v", v_loc)):
                if tuple(t.shape) != shape:
                    raise DimensionError(f"{n} shard must have shape {shape}, got {tuple(t.shape)}")
            return self._forward_ipc(q_loc, k_loc, v_loc)
        return self._forward_p2p(q_loc, k_loc, v_loc)

    def capture(self, q_loc, k_loc, v_loc, warmup=2) -> Partial:
        """Record one forward over these input tensors as a CUDA graph; every
        later call with the same three tensors (same storage: refill them in
        place) replays it -- one graph launch of host work per forward instead
        of the step loop's ~10 launches per step, which at small S outruns
        the GPU (32K tokens on 8 ranks: ~2.8 ms of Python per forward against
        ~1.3 ms of device work).  The flags' sequence values are epoch-relative
        (tr_flag_*_rel, advanced on the device by the graph's last node), so
        replays need no host bookkeeping.  Collective: every rank captures at
        the same call, after ``warmup`` eager forwards.  ipc / fused
        transports, or one rank; the NCCL transport is not captured."""
        if self.P > 1 and self.transport not in ("ipc", "fused"):
            raise ConfigError("capture() needs the ipc or fused transport (or a single rank)")
        for _ in range(warmup):
            self._forward(q_loc, k_loc, v_loc)
        torch.cuda.synchronize(self.device)
        was, self.record_timeline = self.record_timeline, False
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=self.device)
        try:
            with torch.cuda.device(self.device), torch.cuda.graph(g, stream=side):
                self._forward(q_loc, k_loc, v_loc)
        finally:
            self.record_timeline = was
        self._graph = (g, _ptrs(q_loc, k_loc, v_loc))
        return Partial(self.acc_out, self.acc_lse)

    def _forward_p2p(self, q_loc, k_loc, v_loc) -> Partial:
        shape = (self.local_rows, self.H, self.D)
        for n, t in (("q", q_loc), ("k", k_loc), ("v", v_loc)):
            if tuple(t.shape) != shape:
                raise DimensionError(f"{n} shard must have shape {shape}, got {tuple(t.shape)}")
        c, rank = self.c, self.rank
        local_layout = self.prog[0].q_layout
        if not self.direct_first:
            self.ops.init_(self.acc_out, self.acc_lse)
        pending, pending_out = [], None
        self.timeline = []
        for st in self.prog:
            i = st.step
            ev = {}
            _nvtx_push(f"tokenring step {i}")
            if self.record_timeline:
                ev["start"] = self.ops.event()
                self.ops.record(ev["start"])
            for r in pending:
                r.wait()
            if self.record_timeline:
                ev["comm_ready"] = self.ops.event()
                self.ops.record(ev["comm_ready"])
            if pending_out:
                self._merge_returned(pending_out, local_layout)
            sends, recvs = [], []
            cur = self.qbuf[st.q_slot] if st.q_slot >= 0 else q_loc
            kst, vst, kv_lay, kv_local = self._kv_store(st, k_loc, v_loc)
            for dst, ids, from_home in st.send_q:
                src_buf, src_layout = (q_loc, local_layout) if from_home else (cur, st.q_layout)
                a, b = _rows(src_layout, ids, c)
                sends.append((dst, src_buf[a:b]))
            nxt = self._next_layout(rank, i) if st.recv_q else ()
            for src, ids in st.recv_q:
                a, b = _rows(nxt, ids, c)
                recvs.append((src, self.qbuf[(i + 1) % 2][a:b]))
            if st.send_out is not None:
                prev_layout = self.prog[i - 1].q_layout
                a, b = _rows(prev_layout, st.send_out[1], c)
                ob, lb = self.obuf[(i - 1) % 2], self.lbuf[(i - 1) % 2]
                ls = self.lse_send.view(-1)[: self.H * (b - a)].view(self.H, b - a)
                ls.copy_(lb[:, a:b])
                sends.append((st.send_out[0], ob[a:b]))
                sends.append((st.send_out[0], ls))
            pending_out = None
            if st.recv_out:
                if len(st.recv_out) != 1:
                    raise ScheduleError(f"step {i} rank {rank}: more than one return per step")
                src, ids = st.recv_out[0]
                n = len(ids) * c
                lr = self.lse_recv.view(-1)[: self.H * n].view(self.H, n)
                recvs.append((src, self.out_recv[:n]))
                recvs.append((src, lr))
                pending_out = (ids, self.out_recv[:n], lr)
            if st.send_kv is not None:          # hybrid: KV to the next node's rank
                a, b = _rows(kv_lay, st.send_kv[1], c)
                sends.append((st.send_kv[0], kst[a:b]))
                sends.append((st.send_kv[0], vst[a:b]))
            if st.recv_kv is not None:
                kb, vb = self.kvbuf[self.prog[i + 1].kv_store % 2]
                n = len(st.recv_kv[1]) * c
                recvs.append((st.recv_kv[0], kb[:n]))
                recvs.append((st.recv_kv[0], vb[:n]))
            pending = self._comm(sends, recvs)
            if st.q_ids:
                q_segs = []
                for a in st.q_ids:
                    r0, _ = _rows(st.q_layout, (a,), c)
                    q_segs.append((r0, c, self.sched.chunks[a].start))
                kv_segs = self._kv_segs(st, kv_local)
                buf = i % 2
                if self.record_timeline:
                    ev["attn_start"] = self.ops.event()
                    self.ops.record(ev["attn_start"])
                first = i == 0 and self.direct_first
                self.ops.attention(cur, kst, vst, q_segs, kv_segs, self.causal,
                                   self.acc_out if first else self.obuf[buf],
                                   self.acc_lse if first else self.lbuf[buf])
                if self.record_timeline:
                    ev["attn_end"] = self.ops.event()
                    self.ops.record(ev["attn_end"])
                    ev["attn_flops"] = self.step_flops(st)
                if st.accumulate and not first:
                    for a in st.q_ids:
                        r0, r1 = _rows(st.q_layout, (a,), c)
                        l0 = self.part.local_offset(rank, self.sched.chunks[a].start)
                        self.ops.merge_(self.acc_out[l0:l0 + c], self.acc_lse[:, l0:l0 + c],
                                        self.obuf[buf][r0:r1], self.lbuf[buf][:, r0:r1])
            if self.record_timeline:
                ev["computed"] = self.ops.event()
                self.ops.record(ev["computed"])
                self.timeline.append(ev)
            _nvtx_pop()
        for r in pending:
            r.wait()
        if pending_out:
            self._merge_returned(pending_out, local_layout)
        return Partial(self.acc_out, self.acc_lse)

    def _next_layout(self, dst, step):
        """Row layout of ``dst``'s traveling-Q buffer after the messages of
        ``step`` land (all Q chunks sent to it that step, in start order) --
        what its own ``compile_rank`` derives."""
        key = (dst, step)
        if key not in self._layouts:
            plan = self.sched.all_plans()[step]
            ids = [a for src in range(self.P) for m in plan.sends[src]
                   if m.dst == dst and m.kind is MsgKind.Q_BLOCK for a in m.chunk_ids]
            self._layouts[key] = tuple(sorted(ids, key=lambda a: self.sched.chunks[a].start))
        return self._layouts[key]

    def step_flops(self, st) -> int:
        """Algorithmic flops of one step's launch (ref engine.py:170-173)."""
        from .engine import compute_flops
        plan = self.sched.all_plans()[st.step]
        ch = self.sched.chunks
        return sum(compute_flops(cp.mask, ch[cp.q_chunk].tokens, ch[cp.kv_chunk].tokens,
                                 self.H, self.D) for cp in plan.computes[self.rank])

    def _merge_returned(self, pending_out, local_layout):
        ids, out, lse = pending_out
        c = self.c
        for j, a in enumerate(ids):
            if self.sched.chunks[a].home != self.rank:
                raise ScheduleError(f"rank {self.rank}: returned chunk {a} homes elsewhere")
            l0 = self.part.local_offset(self.rank, self.sched.chunks[a].start)
            self.ops.merge_(self.acc_out[l0:l0 + c], self.acc_lse[:, l0:l0 + c],
                            out[j * c:(j + 1) * c], lse[:, j * c:(j + 1) * c])


def token_ring_attention(q_loc, k_loc, v_loc, seq_len, causal=True, group=None) -> Partial:
    """Functional form: one TokenRing forward over ``group`` (all ranks call it)."""
    h, d = q_loc.shape[1], q_loc.shape[2]
    return TokenRingAttention(seq_len, h, d, causal, group, device=q_loc.device)(q_loc, k_loc, v_loc)


def check_world(seq_len, causal, world):
    """ConfigError early if the sequence does not split over ``world`` ranks."""
    need = 2 * world if causal else world
    if seq_len % need:
        raise ConfigError(f"seq_len {seq_len} must be divisible by {need}")
