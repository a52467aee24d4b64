"""The multi-process runner with one process per DISTINCT GPU -- the
deployment shape of SURVEY 8(e) -- for every transport (NCCL P2P, copy
engines into IPC-mapped peer memory, the fused epilogue push over NVLink)
and every schedule the runner carries (zigzag TokenRing on the reference's
ring route and on the direct route, non-causal TokenRing, and the Ring
Attention KV rotation of ref engine.py:203-230), checked rank by rank
against the oracle's execute of the same schedule.

Skips cleanly on a box with fewer than 2 GPUs (every gpurun call of this
round had one); the single-GPU rehearsals of the same code paths are
tests/test_gpu_ring_ipc.py (processes sharing cuda:0) and
tests/test_ring_gloo.py (host logic over gloo)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import schedule as osch
from oracle import splitmix

pytestmark = pytest.mark.gpu

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0

_reap = []


@pytest.fixture(autouse=True)
def _kill_workers():
    yield
    while _reap:
        p = _reap.pop()
        if p.is_alive():
            p.kill()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SEEDS = (31, 32)


def _worker(rank, world, port, S, H, D, causal, route, transport, schedule, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl" if transport == "nccl" else "gloo", rank=rank,
                            world_size=world, **({"device_id": dev} if transport == "nccl" else {}))
    try:
        from paper_2412_20501_b200 import rng
        from paper_2412_20501_b200.ring import TokenRingAttention
        runner = TokenRingAttention(S, H, D, causal=causal, device=dev, transport=transport,
                                    route=route, schedule=schedule)
        outs = []
        for sd in SEEDS:
            res = runner(*rng.local_inputs(sd, runner.part, rank, H, D, device=dev))
            outs.append((res.out.clone(), res.lse.clone()))
        torch.cuda.synchronize()
        q_out.put((rank, [(o.double().cpu().numpy(), l.double().cpu().numpy()) for o, l in outs]))
        if hasattr(runner, "peer"):
            runner.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


CASES = [(w, t, s, r, c) for w in (2, 4, 8) for t in ("nccl", "ipc", "fused")
         for s, r, c in (("token-ring", "ring", True), ("token-ring", "direct", True),
                         ("token-ring", "ring", False), ("ring", "ring", True))
         if not (r == "direct" and w < 3)]


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs (one process per device)")
@pytest.mark.parametrize("world,transport,schedule,route,causal", CASES)
def test_runner_on_distinct_devices(world, transport, schedule, route, causal):
    if world > NGPU:
        pytest.skip(f"needs {world} GPUs, box has {NGPU}")
    if transport != "nccl":
        for a in range(world):
            for b in range(world):
                if a != b and not torch.cuda.can_device_access_peer(a, b):
                    pytest.skip(f"no P2P path between GPU {a} and GPU {b}")
    S, H, D = 1024 * world, 2, 128
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, S, H, D, causal, route, transport,
                                               schedule, q_out)) for r in range(world)]
    for p in procs:
        p.start()
    _reap.extend(procs)
    res = dict(q_out.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    if schedule == "ring":
        sched = osch.ring(world, S, H, D, causal)
    else:
        sched = osch.zigzag_token_ring(world, S, H, D) if causal else osch.token_ring(world, S, H, D)
    for call, sd in enumerate(SEEDS):
        q, k, v = (splitmix.to_bf16_f64(x) for x in splitmix.attention_inputs(sd, S, H, D))
        ref = osch.execute(sched, q, k, v)
        for r in range(world):
            out, lse = res[r][call]
            assert np.abs(out - ref[r][0]).max() <= 2e-2, (r, call)
            fin = np.isfinite(ref[r][1])
            assert np.array_equal(np.isfinite(lse), fin)
            assert np.abs(lse[fin] - ref[r][1][fin]).max() <= 1e-3, (r, call)
