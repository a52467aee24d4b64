"""End-to-end GPU parity of the schedule executor and the ring runner against
the reference (golden fixtures from ringsim.engine.execute) and the oracle.
Tolerances: out max-abs 2e-2, lse max-abs 1e-3 on bf16-rounded inputs."""

import numpy as np
import pytest
import torch

from oracle import kernels as ok
from oracle import partition as opart
from oracle import schedule as osch
from oracle import splitmix

pytestmark = pytest.mark.gpu


def dev(x):
    return torch.as_tensor(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).cuda()


def close(got_out, got_lse, ref_out, ref_lse, name=""):
    go = got_out.double().cpu().numpy() if isinstance(got_out, torch.Tensor) else got_out
    gl = got_lse.double().cpu().numpy() if isinstance(got_lse, torch.Tensor) else got_lse
    fin = np.isfinite(ref_lse)
    assert np.array_equal(np.isfinite(gl), fin), name
    assert np.abs(gl[fin] - ref_lse[fin]).max() <= 1e-3, (name, np.abs(gl[fin] - ref_lse[fin]).max())
    assert np.abs(go - ref_out).max() <= 2e-2, (name, np.abs(go - ref_out).max())


def test_execute_matches_reference_golden(golden_execute):
    import paper_2412_20501_b200 as tr
    meta, arr = golden_execute
    for m in meta:
        kind, p, s, h, d, causal = m["args"][:6]
        nodes = m["args"][6] if len(m["args"]) > 6 else 1
        sc = tr.build_schedule(kind, p, s, h, d, causal if kind == "ring" else None, nodes=nodes)
        q, k, v = splitmix.attention_inputs(m["seed"], s, h, d)
        qb, kb, vb = (splitmix.to_bf16_f64(x) for x in (q, k, v))
        outs, trace = tr.execute(sc, dev(qb), dev(kb), dev(vb))
        torch.cuda.synchronize()
        ref = osch.execute(osch.by_name(*m["args"]), qb, kb, vb)
        for r in range(p):
            if m["bf16"]:       # golden itself was computed on bf16-rounded inputs
                close(outs[r].out, outs[r].lse, arr[f"{m['name']}__out{r}"],
                      arr[f"{m['name']}__lse{r}"], m["name"])
            close(outs[r].out, outs[r].lse, ref[r][0], ref[r][1], m["name"])
        assert sum(c.flops for c in trace.computes) == osch.flops(osch.by_name(*m["args"]), h, d)


@pytest.mark.parametrize("P,S,H,D,route", [(2, 4096, 8, 64, "ring"), (4, 4096, 4, 128, "ring"),
                                           (8, 8192, 2, 128, "ring"), (1, 2048, 4, 128, "ring"),
                                           (8, 8192, 2, 128, "direct"), (5, 5120, 2, 64, "direct")])
def test_execute_zigzag_vs_dense_oracle(P, S, H, D, route):
    import paper_2412_20501_b200 as tr
    q, k, v = (splitmix.to_bf16_f64(x) for x in splitmix.attention_inputs(3 + P, S, H, D))
    sc = tr.build_zigzag_token_ring(P, S, H, D, route=route)
    outs, _ = tr.execute(sc, dev(q), dev(k), dev(v))
    merged = tr.global_reorder(outs, sc.partition)
    torch.cuda.synchronize()
    ref_o, ref_l = ok.dense_attention(q, k, v, causal=True)
    close(merged.out, merged.lse, ref_o, ref_l, f"zigzag P={P} {route}")


def test_config1_token_ring_p2():
    """BASELINE config 1: TokenRing, 2 simulated ranks, S=4096, H=8, D=64,
    non-causal, seed 0 -- GPU execute vs the oracle's execute."""
    import paper_2412_20501_b200 as tr
    S, H, D = 4096, 8, 64
    q, k, v = (splitmix.to_bf16_f64(x) for x in splitmix.attention_inputs(0, S, H, D))
    sc = tr.build_token_ring(2, S, H, D)
    outs, _ = tr.execute(sc, dev(q), dev(k), dev(v))
    torch.cuda.synchronize()
    ref = osch.execute(osch.token_ring(2, S, H, D), q, k, v)
    for r in range(2):
        close(outs[r].out, outs[r].lse, ref[r][0], ref[r][1], f"cfg1 rank {r}")


def test_ring_runner_single_rank_equals_dense():
    """TokenRingAttention with world size 1 (no process group) = one causal block."""
    from paper_2412_20501_b200 import rng
    from paper_2412_20501_b200.ring import TokenRingAttention
    S, H, D = 4096, 4, 128
    q, k, v = rng.attention_inputs(5, S, H, D)
    res = TokenRingAttention(S, H, D, causal=True)(q, k, v)
    torch.cuda.synchronize()
    qn, kn, vn = (splitmix.to_bf16_f64(x) for x in splitmix.attention_inputs(5, S, H, D))
    assert np.array_equal(q.double().cpu().numpy(), qn)
    ref_o, ref_l = ok.dense_attention(qn, kn, vn, causal=True)
    close(res.out, res.lse, ref_o, ref_l, "ring P=1")


def test_ring_runner_single_rank_graph_replay():
    """capture() on one rank: replays of the CUDA graph with the static inputs
    refilled in place equal eager forwards of the same inputs, bit for bit."""
    from paper_2412_20501_b200 import rng
    from paper_2412_20501_b200.ring import TokenRingAttention
    S, H, D = 4096, 4, 128
    ins = [rng.attention_inputs(sd, S, H, D) for sd in (5, 6)]
    eager = TokenRingAttention(S, H, D, causal=True)
    want = []
    for t in ins:
        r = eager(*t)
        want.append((r.out.clone(), r.lse.clone()))
    runner = TokenRingAttention(S, H, D, causal=True)
    static = [t.clone() for t in ins[0]]
    runner.capture(*static)
    for i in (1, 0, 1):
        for d, s_ in zip(static, ins[i]):
            d.copy_(s_)
        r = runner(*static)
        assert torch.equal(r.out, want[i][0]) and torch.equal(r.lse, want[i][1]), i


def test_bench_e2e_pipeline_outputs():
    """bench.py's end-to-end leg (head groups, edge pieces, copy streams,
    double-buffered staging) hands back in pinned host memory exactly what
    one runner over all heads computes on the device."""
    import bench
    from paper_2412_20501_b200 import rng
    from paper_2412_20501_b200.ring import TokenRingAttention
    S, H, D = 4096, 8, 128
    q, k, v = rng.attention_inputs(11, S, H, D)
    ref = TokenRingAttention(S, H, D, causal=True)(q, k, v)
    want_o, want_l = ref.out.to(torch.bfloat16).cpu(), ref.lse.cpu()
    ms, outs = bench.e2e_pipelined(lambda n: TokenRingAttention(S, n, D, causal=True),
                                   q, k, v, 3, lambda: None, lambda x: x, 2, edge=1,
                                   return_outputs=True)
    assert ms > 0
    # groups of 4 heads; the run's first and last groups split off 1-head pieces
    assert set(outs) == {(0, 4), (4, 8), (0, 1), (1, 4), (4, 7), (7, 8)}
    for (a, b), slots in outs.items():
        for o, l in slots:
            if not l.abs().sum():          # a parity this range never ran at
                continue
            assert torch.equal(o, want_o[:, a:b]), (a, b)
            assert torch.equal(l, want_l[a:b]), (a, b)


def test_block_attention_api_and_errors():
    import paper_2412_20501_b200 as tr
    q, k, v = splitmix.attention_inputs(42, 4, 2, 3)
    p = tr.block_attention(q, k, v)
    # bf16-rounded inputs on both sides
    ro, rl = ok.attention_block(*(splitmix.to_bf16_f64(x) for x in (q, k, v)))
    close(p.out, p.lse, ro, rl, "kat42")
    with pytest.raises(tr.DimensionError):
        tr.block_attention(q, k[:, :1], v)
    bad = q.copy()
    bad[0, 0, 0] = np.nan
    with pytest.raises(tr.InputError):
        tr.block_attention(bad, k, v)
    e = tr.Partial.empty(4, 2, 3)
    m = tr.merge_partial(e, p)          # empty accumulator is an exact identity
    assert torch.equal(m.lse, p.lse) and torch.equal(m.out, p.out.float())
    with pytest.raises(tr.DimensionError):
        tr.merge_partial(tr.Partial.empty(3, 2, 3), p)
