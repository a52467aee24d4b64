"""The multi-process TokenRing runner (paper_2412_20501_b200.ring) at
world_size 2 and 4 over gloo on CPU.  The device ops are replaced by the
float64 oracle (test-only injection, tests/cpu_ops.py) so what is checked
here is the host side: rank programs, buffer layouts, Q-forward and
OUT-reverse P2P traffic and merge bookkeeping."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import kernels as ok
from oracle import partition as opart
from oracle import schedule as osch
from oracle import splitmix


_reap = []     # workers of the current test; killed if a test fails mid-way


@pytest.fixture(autouse=True)
def _kill_workers():
    yield
    while _reap:
        p = _reap.pop()
        if p.is_alive():
            p.kill()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, S, H, D, causal, seed, result_q, route="ring", nodes=1,
            schedule="token-ring"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cpu_ops import OracleOps
        from paper_2412_20501_b200.ring import TokenRingAttention
        runner = TokenRingAttention(S, H, D, causal=causal, ops=OracleOps(), device="cpu",
                                    route=route, nodes=nodes, schedule=schedule)
        q, k, v = (splitmix.to_bf16_f64(x) for x in splitmix.attention_inputs(seed, S, H, D))
        rng = runner.part.ranges(rank)
        loc = [torch.as_tensor(opart.gather(x, rng), dtype=torch.float32).to(torch.bfloat16)
               for x in (q, k, v)]
        res = runner(*loc)
        result_q.put((rank, res.out.double().numpy(), res.lse.double().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,S,H,D,causal,route", [
    (2, 64, 2, 8, True, "ring"), (4, 128, 2, 8, True, "ring"), (2, 48, 2, 8, False, "ring"),
    (3, 96, 1, 8, True, "ring"),
    # non-reference NVSwitch-aware Q routing: same computes, different messages
    (4, 128, 2, 8, True, "direct"), (5, 160, 1, 8, True, "direct")])
def test_token_ring_gloo(world, S, H, D, causal, route):
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, S, H, D, causal, 11, q_, route))
             for r in range(world)]
    for p in procs:
        p.start()
    _reap.extend(procs)
    res = {}
    for _ in range(world):
        r, o, l = q_.get(timeout=120)
        res[r] = (o, l)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    q, k, v = (splitmix.to_bf16_f64(x) for x in splitmix.attention_inputs(11, S, H, D))
    sched = osch.zigzag_token_ring(world, S, H, D) if causal else osch.token_ring(world, S, H, D)
    ref = osch.execute(sched, q, k, v)
    for r in range(world):
        # bf16 block outputs travel between ranks; accumulators stay float32
        assert np.abs(res[r][0] - ref[r][0]).max() <= 2e-2
        fin = np.isfinite(ref[r][1])
        assert np.array_equal(np.isfinite(res[r][1]), fin)
        assert np.abs(res[r][1][fin] - ref[r][1][fin]).max() <= 1e-3
    g_out, g_lse = opart.reorder([res[r][0] for r in range(world)],
                                 [res[r][1] for r in range(world)], osch.ranges_of(sched, S), S)
    d_out, d_lse = ok.dense_attention(q, k, v, causal)
    assert ok.max_relative_error(g_out, g_lse, d_out, d_lse) <= 2e-2


@pytest.mark.parametrize("nodes,per_node,S", [(2, 2, 64), (2, 3, 96), (3, 2, 96)])
def test_hybrid_gloo(nodes, per_node, S):
    """The reference's multi-node schedule (TokenRing inside a node, KV
    rotated across nodes; ref engine.py:233-303) run by the multi-process
    runner: KV blocks travel at the hand-off steps into the receiver's second
    KV store, per rank the result equals the oracle's execute of the same
    schedule, and the whole equals dense non-causal attention."""
    world, H, D = nodes * per_node, 2, 8
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, S, H, D, False, 13, q_, "ring", nodes))
             for r in range(world)]
    for p in procs:
        p.start()
    _reap.extend(procs)
    res = {}
    for _ in range(world):
        r, o, l = q_.get(timeout=120)
        res[r] = (o, l)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    q, k, v = (splitmix.to_bf16_f64(x) for x in splitmix.attention_inputs(13, S, H, D))
    sched = osch.hybrid(nodes, per_node, S, H, D)
    ref = osch.execute(sched, q, k, v)
    for r in range(world):
        assert np.abs(res[r][0] - ref[r][0]).max() <= 2e-2
        assert np.abs(res[r][1] - ref[r][1]).max() <= 1e-3
    g_out, g_lse = opart.reorder([res[r][0] for r in range(world)],
                                 [res[r][1] for r in range(world)], osch.ranges_of(sched, S), S)
    d_out, d_lse = ok.dense_attention(q, k, v, False)
    assert ok.max_relative_error(g_out, g_lse, d_out, d_lse) <= 2e-2


@pytest.mark.parametrize("world,S,causal", [(2, 64, True), (4, 128, True), (3, 48, False),
                                            (4, 64, False), (5, 80, True)])
def test_ring_attention_gloo(world, S, causal):
    """Ring Attention (KV rotation, ref engine.py:203-230) -- the config-4
    baseline -- on the multi-process runner: contiguous shards, KV blocks
    forwarded to rank+1 every step into the receiver's alternate KV store,
    the causal ring's fully-masked blocks skipped; per rank equal to the
    oracle's execute of the same schedule and, reassembled, to dense
    attention."""
    H, D = 2, 8
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, S, H, D, causal, 17, q_, "ring", 1, "ring"))
             for r in range(world)]
    for p in procs:
        p.start()
    _reap.extend(procs)
    res = {}
    for _ in range(world):
        r, o, l = q_.get(timeout=120)
        res[r] = (o, l)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    q, k, v = (splitmix.to_bf16_f64(x) for x in splitmix.attention_inputs(17, S, H, D))
    sched = osch.ring(world, S, H, D, causal)
    ref = osch.execute(sched, q, k, v)
    for r in range(world):
        assert np.abs(res[r][0] - ref[r][0]).max() <= 2e-2
        fin = np.isfinite(ref[r][1])
        assert np.array_equal(np.isfinite(res[r][1]), fin)
        assert np.abs(res[r][1][fin] - ref[r][1][fin]).max() <= 1e-3
    g_out, g_lse = opart.reorder([res[r][0] for r in range(world)],
                                 [res[r][1] for r in range(world)], osch.ranges_of(sched, S), S)
    d_out, d_lse = ok.dense_attention(q, k, v, causal)
    assert ok.max_relative_error(g_out, g_lse, d_out, d_lse) <= 2e-2


def _worker_capture(rank, world, port, result_q):
    """capture() refuses the NCCL transport (P2P ops of a process group are
    not captured); checked before any device work."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cpu_ops import OracleOps
        from paper_2412_20501_b200.errors import ConfigError
        from paper_2412_20501_b200.ring import TokenRingAttention
        runner = TokenRingAttention(64, 2, 8, causal=True, ops=OracleOps(), device="cpu")
        try:
            runner.capture(None, None, None)
            result_q.put((rank, "no error"))
        except ConfigError as e:
            result_q.put((rank, "ConfigError" if "ipc or fused" in str(e) else str(e)))
    finally:
        dist.destroy_process_group()


def test_capture_refuses_nccl_transport():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_capture, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    _reap.extend(procs)
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert got == {0: "ConfigError", 1: "ConfigError"}, got
