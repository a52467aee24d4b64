"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The fixtures in tests/golden were produced by scripts/make_golden.py from
the reference package itself; the frozen known-answer values are the ones in
the reference's own tests (pkg/tests/test_core.py:36-45,191-198).
"""

import numpy as np
import pytest

from conftest import load_json
from oracle import kernels as ok
from oracle import partition as opart
from oracle import schedule as osch
from oracle import splitmix


def test_splitmix_kats():
    kat = load_json("rng_kats.json")
    assert [int(x) for x in splitmix.hash_draws(42, 0, 4)] == kat["raw_stream_42_4"]
    # SURVEY App. B, hex form
    assert hex(kat["raw_stream_42_4"][0]) == "0xbdd732262feb6e95"
    assert list(splitmix.unit_doubles(42, 0, 4)) == kat["uniform_42_4"]
    q, k, v = splitmix.attention_inputs(42, 4, 2, 3)
    assert list(q[0, 0]) == kat["inputs_42_4_2_3_q0"]
    q, k, v = splitmix.attention_inputs(0, 4096, 8, 64)
    assert list(q[0, 0, :3]) == kat["inputs_0_4096_8_64_q0"]
    assert v[-1, -1, -1] == kat["inputs_0_4096_8_64_vlast"]
    assert k[2048, 3, 17] == kat["inputs_0_4096_8_64_k_mid"]


def test_splitmix_row_windows_match_full_stream():
    q, k, v = splitmix.attention_inputs(5, 40, 3, 8)
    for which, full in enumerate((q, k, v)):
        rows = splitmix.attention_rows(5, 40, 3, 8, which, 13, 9)
        assert np.array_equal(rows, full[13:22])


def test_bf16_rounding_is_rne():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -0.3, 1e-30, 0.0])
    got = splitmix.to_bf16_f64(x)
    assert got[0] == 1.0
    assert got[1] == 1.0          # tie -> even
    assert got[2] == 1.0 + 2 ** -7
    assert abs(got[3] + 0.3) < 2 ** -9
    import torch
    t = torch.tensor(x, dtype=torch.float64).to(torch.float32).to(torch.bfloat16)
    assert np.array_equal(got, t.to(torch.float64).numpy())


def test_known_answers_seed42():
    q, k, v = splitmix.attention_inputs(42, 4, 2, 3)
    out, lse = ok.attention_block(q, k, v)
    assert lse[0, 0] == pytest.approx(1.144157354277393, abs=1e-13)
    assert out[0, 0, 0] == pytest.approx(-0.17376816644158208, abs=1e-13)
    assert out[3, 1, 2] == pytest.approx(-0.08708629600115192, abs=1e-13)
    out, lse = ok.dense_attention(q, k, v, causal=True)
    assert lse[0, 0] == pytest.approx(-0.18658740071149307, abs=1e-13)
    assert out[2, 1, 1] == pytest.approx(-0.11089228754240948, abs=1e-13)


def test_closed_forms():
    one = np.ones((1, 1, 1))
    out, lse = ok.attention_block(one, one, one)
    assert out[0, 0, 0] == 1.0 and lse[0, 0] == 1.0
    q = np.array([[[1.0, 0.5]]])
    key = np.array([0.25, -0.75])
    k = np.stack([key, key])[:, None, :]
    v = np.stack([np.array([2.0, -4.0]), np.array([6.0, 8.0])])[:, None, :]
    out, lse = ok.attention_block(q, k, v)
    np.testing.assert_allclose(out[0, 0], [4.0, 2.0], rtol=1e-15)
    np.testing.assert_allclose(lse[0, 0], (q[0, 0] @ key) / np.sqrt(2) + np.log(2), rtol=1e-15)


def test_attention_golden(golden_kernels):
    meta, arr = golden_kernels
    for m in meta:
        n = m["name"]
        q, k, v = (arr[f"{n}__{x}"].astype(np.float64) for x in "qkv")
        kind = {"none": ok.MASK_NONE, "fully_masked": ok.MASK_FULL,
                "causal": ok.MASK_CAUSAL}[m["mask"]]
        out, lse = ok.attention_block(q, k, v, kind, m["q_offset"], m["k_offset"])
        ref_out, ref_lse = arr[f"{n}__out"], arr[f"{n}__lse"]
        np.testing.assert_allclose(out, ref_out, rtol=1e-12, atol=1e-13, err_msg=n)
        fin = np.isfinite(ref_lse)
        assert np.array_equal(np.isfinite(lse), fin), n
        np.testing.assert_allclose(lse[fin], ref_lse[fin], rtol=1e-12, atol=1e-13, err_msg=n)


def test_merge_golden(golden_merge):
    names, arr = golden_merge
    for n in names:
        out, lse = ok.merge_state(arr[f"{n}__acc_out"], arr[f"{n}__acc_lse"],
                                  arr[f"{n}__blk_out"], arr[f"{n}__blk_lse"])
        np.testing.assert_allclose(out, arr[f"{n}__out"], rtol=1e-14, atol=1e-15, err_msg=n)
        ref = arr[f"{n}__lse"]
        fin = np.isfinite(ref)
        assert np.array_equal(np.isfinite(lse), fin)
        np.testing.assert_allclose(lse[fin], ref[fin], rtol=1e-14, err_msg=n)
    # exact identities (ref test_core.py:108-131)
    o, l = ok.merge_state(np.array([[[1.0, -2.25]]]), np.zeros((1, 1)),
                          np.array([[[3.0, 0.75]]]), np.zeros((1, 1)))
    assert np.array_equal(o, np.array([[[2.0, -0.75]]])) and l[0, 0] == np.log(2)


def _build(kind, p, s, h, d, causal, nodes=1):
    return osch.by_name(kind, p, s, h, d, causal, nodes)


def test_schedules_golden(golden_schedules):
    for g in golden_schedules:
        kind, p, s, h, d, causal = g["args"][:6]
        sc = _build(*g["args"])
        assert sc == g["schedule"], g["args"]
        rr = osch.ranges_of(sc, s)
        assert [list(map(list, x)) for x in rr] == g["ranges"]
        assert list(opart.causal_pairs(rr)) == g["causal_work"]
        assert osch.flops(sc, h, d) == g["flops_total"]


def test_execute_golden(golden_execute):
    meta, arr = golden_execute
    for m in meta:
        kind, p, s, h, d, causal = m["args"][:6]
        if s * h * d > 300_000:
            continue       # large fixtures are for the GPU tests
        sc = _build(*m["args"])
        q, k, v = splitmix.attention_inputs(m["seed"], s, h, d)
        if m["bf16"]:
            q, k, v = (splitmix.to_bf16_f64(x) for x in (q, k, v))
        outs = osch.execute(sc, q, k, v)
        for r in range(p):
            np.testing.assert_allclose(outs[r][0], arr[f"{m['name']}__out{r}"], rtol=1e-12,
                                       atol=1e-13)
            np.testing.assert_allclose(outs[r][1], arr[f"{m['name']}__lse{r}"], rtol=1e-12,
                                       atol=1e-13)
        g_out, g_lse = opart.reorder([outs[r][0] for r in range(p)],
                                     [outs[r][1] for r in range(p)], osch.ranges_of(sc, s), s)
        assert ok.max_relative_error(g_out, g_lse, arr[f"{m['name']}__dense_out"],
                                     arr[f"{m['name']}__dense_lse"]) <= 1e-10


def test_zigzag_structure_rules():
    # identical per-rank work each step; only chunk 0 pruned
    for p in (2, 3, 4, 8):
        sc = osch.zigzag_token_ring(p, 16 * p, 1, 2)
        c = 8
        for step in sc["steps"]:
            works = []
            for r in range(p):
                pairs = 0
                for a, b, m, qo, ko, _ in step[r]["computes"]:
                    pairs += c * c if m == "none" else c * (c + 1) // 2
                works.append(pairs)
            assert len(set(works)) == 1
        for i, step in enumerate(sc["steps"][:-1]):
            for r in range(p):
                q_sends = [s for s in step[r]["sends"] if s[1] == "q_block"]
                assert len(q_sends) == 1
                assert 0 < len(q_sends[0][2]) <= 2
                assert 2 * p - 1 - ((r - i) % p) in q_sends[0][2]


def test_reference_compiled_kernels_agree_when_built(golden_kernels):
    """oracle/_ref holds the reference's Cython kernels compiled from
    /root/reference (oracle/Makefile); cross-check when it is present."""
    from oracle import ref_kernels
    mod = ref_kernels.load()
    if mod is None:
        pytest.skip("oracle/_ref not built")
    meta, arr = golden_kernels
    for m in meta:
        n = m["name"]
        q, k, v = (np.ascontiguousarray(arr[f"{n}__{x}"], dtype=np.float64) for x in "qkv")
        kind = {"none": 0, "fully_masked": 1, "causal": 2}[m["mask"]]
        out, lse = mod.attention_block(q, k, v, kind, m["q_offset"], m["k_offset"])
        np.testing.assert_allclose(out, arr[f"{n}__out"], rtol=1e-11, atol=1e-12)
