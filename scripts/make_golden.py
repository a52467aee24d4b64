"""Generate tests/golden/* by importing the reference ``ringsim`` package.

Run in the build container only (``/root/reference`` does not exist on the GPU
box); the committed fixtures are what the tests read:

    RINGSIM_KERNELS=python python scripts/make_golden.py [/root/reference/pkg/src]

Everything here is produced by the reference's own public API (rng,
block_attention, merge_partial, the schedule builders, execute,
comm_volume, trace_from_schedule).  The numpy backend is forced so the
vectors are the reference's ``_kernels_ref`` arithmetic.
"""

import json
import os
import sys

import numpy as np

os.environ.setdefault("RINGSIM_KERNELS", "python")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
SRC = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, SRC)

import ringsim  # noqa: E402
from ringsim import engine, partition, rng  # noqa: E402
from ringsim.core import MaskSpec  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
os.makedirs(OUT, exist_ok=True)


def to_bf16_f64(x):
    f = np.ascontiguousarray(x, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    b = ((b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def canon_mask(m):
    return [m.kind.value, int(m.q_offset), int(m.k_offset)]


def canon_plan(plan, ranks):
    out = []
    for r in range(ranks):
        out.append({
            "computes": [[cp.q_chunk, cp.kv_chunk, *canon_mask(cp.mask), bool(cp.accumulate)]
                         for cp in plan.computes[r]],
            "sends": [[m.dst, m.kind.value, list(m.chunk_ids), int(m.payload_elements)]
                      for m in plan.sends[r]],
            "merges": [[mp.src, list(mp.chunk_ids)] for mp in plan.merges[r]],
        })
    return out


def canon(s):
    return {"kind": s.kind, "ranks": s.ranks, "causal": bool(s.causal),
            "chunks": [[c.id, c.start, c.stop, c.home] for c in s.chunks],
            "steps": [canon_plan(p, s.ranks) for p in s.steps],
            "final": canon_plan(s.final_phase, s.ranks) if s.final_phase else None}


def rng_kats():
    q, k, v = rng.attention_inputs(0, 4096, 8, 64)
    return {
        "raw_stream_42_4": [int(x) for x in rng.raw_stream(42, 4)],
        "uniform_42_4": [float(x) for x in rng.uniform(42, (4,))],
        "inputs_42_4_2_3_q0": [float(x) for x in rng.attention_inputs(42, 4, 2, 3)[0][0, 0]],
        "inputs_0_4096_8_64_q0": [float(x) for x in q[0, 0, :3]],
        "inputs_0_4096_8_64_vlast": float(v[-1, -1, -1]),
        "inputs_0_4096_8_64_k_mid": float(k[2048, 3, 17]),
    }


KERNEL_CASES = [
    # name, seed, tq, tk, H, D, mask, q_off, k_off, low, high, bf16
    ("kat42", 42, 4, 4, 2, 3, "none", 0, 0, -1.0, 1.0, False),
    ("kat42_causal", 42, 4, 4, 2, 3, "causal", 0, 0, -1.0, 1.0, False),
    ("agree_none", 5, 12, 12, 3, 7, "none", 0, 0, -3.0, 3.0, False),
    ("agree_full", 5, 12, 12, 3, 7, "fully_masked", 0, 0, -3.0, 3.0, False),
    ("agree_causal", 5, 12, 12, 3, 7, "causal", 0, 0, -3.0, 3.0, False),
    ("agree_causal_8_4", 5, 12, 12, 3, 7, "causal", 8, 4, -3.0, 3.0, False),
    ("agree_causal_0_100", 5, 12, 12, 3, 7, "causal", 0, 100, -3.0, 3.0, False),
    # bf16-rounded inputs at the GPU kernel's head dims (parity fixtures)
    ("bf16_d64_none", 11, 200, 328, 2, 64, "none", 0, 0, -1.0, 1.0, True),
    ("bf16_d64_causal", 12, 256, 256, 2, 64, "causal", 0, 0, -1.0, 1.0, True),
    ("bf16_d128_none", 13, 256, 384, 2, 128, "none", 0, 0, -1.0, 1.0, True),
    ("bf16_d128_causal", 14, 384, 384, 2, 128, "causal", 0, 0, -1.0, 1.0, True),
    ("bf16_d128_causal_off", 15, 192, 320, 2, 128, "causal", 300, 100, -1.0, 1.0, True),
    ("bf16_d128_ragged", 16, 77, 133, 3, 128, "causal", 60, 0, -1.0, 1.0, True),
    ("bf16_d128_maskall", 17, 64, 64, 1, 128, "causal", 0, 500, -1.0, 1.0, True),
    ("bf16_d16_none", 18, 40, 24, 2, 16, "none", 0, 0, -1.0, 1.0, True),
]


def kernel_cases():
    arrs = {}
    meta = []
    for name, seed, tq, tk, h, d, mask, qo, ko, lo, hi, bf in KERNEL_CASES:
        n = max(tq, tk)
        q, k, v = rng.attention_inputs(seed, n, h, d, low=lo, high=hi)
        q, k, v = q[:tq], k[:tk], v[:tk]
        if bf:
            q, k, v = to_bf16_f64(q), to_bf16_f64(k), to_bf16_f64(v)
        spec = {"none": MaskSpec.none(), "fully_masked": MaskSpec.fully_masked(),
                "causal": MaskSpec.causal(qo, ko)}[mask]
        p = ringsim.block_attention(q, k, v, spec)
        store = (lambda x: x.astype(np.float32)) if bf else (lambda x: x)  # bf16 is exact in fp32
        for key, val in (("q", store(q)), ("k", store(k)), ("v", store(v)),
                         ("out", p.out), ("lse", p.lse)):
            arrs[f"{name}__{key}"] = val
        meta.append({"name": name, "seed": seed, "tq": tq, "tk": tk, "heads": h, "dim": d,
                     "mask": mask, "q_offset": qo, "k_offset": ko, "low": lo, "high": hi,
                     "bf16": bf})
    return arrs, meta


def merge_cases():
    arrs = {}
    a_out = rng.uniform(1, (6, 2, 3), -3, 3)
    a_lse = rng.uniform(2, (2, 6), -5, 5)
    b_out = rng.uniform(3, (6, 2, 3), -3, 3)
    b_lse = rng.uniform(4, (2, 6), -5, 5)
    a_lse[0, 0] = -np.inf
    a_out[0, 0, :] = 0.0
    b_lse[1, 3] = -np.inf
    b_out[3, 1, :] = 0.0
    b_lse[0, 5] = -np.inf
    a_lse[0, 5] = -np.inf
    a_out[5, 0, :] = 0.0
    b_out[5, 0, :] = 0.0
    cases = {"mixed": (a_out, a_lse, b_out, b_lse),
             "gap800": (np.ones((1, 1, 1)), np.array([[800.0]]),
                        np.full((1, 1, 1), 2.0), np.array([[-800.0]])),
             "dyadic": (np.array([[[1.0, -2.25]]]), np.zeros((1, 1)),
                        np.array([[[3.0, 0.75]]]), np.zeros((1, 1)))}
    # larger case at the GPU kernel's head dim
    t, h, d = 96, 4, 128
    ao = rng.uniform(21, (t, h, d), -3, 3)
    al = rng.uniform(22, (h, t), -6, 6)
    bo = to_bf16_f64(rng.uniform(23, (t, h, d), -3, 3))
    bl = rng.uniform(24, (h, t), -6, 6)
    drop_a = rng.uniform(25, (h, t)) < 0.2
    drop_b = rng.uniform(26, (h, t)) < 0.2
    al = np.where(drop_a, -np.inf, al)
    ao = np.where(drop_a.T[:, :, None], 0.0, ao)
    bl = np.where(drop_b, -np.inf, bl)
    bo = np.where(drop_b.T[:, :, None], 0.0, bo)
    cases["d128"] = (ao, al, bo, bl)
    for name, (ao, al, bo, bl) in cases.items():
        m = ringsim.merge_partial(ringsim.Partial(ao, al), ringsim.Partial(bo, bl))
        for key, val in (("acc_out", ao), ("acc_lse", al), ("blk_out", bo), ("blk_lse", bl),
                         ("out", m.out), ("lse", m.lse)):
            arrs[f"{name}__{key}"] = val
    return arrs, list(cases)


SCHED_SMALL = []
for p in (1, 2, 3, 4, 8):
    SCHED_SMALL.append(("ring", p, 16 * p, 2, 4, False))
    SCHED_SMALL.append(("ring", p, 16 * p, 2, 4, True))
    SCHED_SMALL.append(("token-ring", p, 16 * p, 2, 4, False))
for p in (1, 2, 3, 4, 8, 16):
    SCHED_SMALL.append(("zigzag-token-ring", p, 8 * p, 2, 4, True))
# evaluation-scale metadata (BASELINE configs 1, 3, 5 and the volume tests)
SCHED_SMALL += [
    ("token-ring", 2, 4096, 8, 64, False),
    ("zigzag-token-ring", 8, 131072, 32, 128, True),
    ("zigzag-token-ring", 4, 131072, 32, 128, True),
    ("zigzag-token-ring", 2, 131072, 32, 128, True),
    ("zigzag-token-ring", 8, 1048576, 64, 128, True),
    ("ring", 8, 131072, 32, 128, True),
    ("token-ring", 4, 24000, 32, 128, False),
    ("ring", 4, 24000, 32, 128, False),
]
# hybrid (TokenRing inside a node, KV rotation across nodes): args carry nodes
SCHED_SMALL += [("hybrid", m * g, 16 * m * g, 2, 4, False, m)
                for m, g in ((1, 1), (1, 4), (2, 1), (2, 2), (2, 4), (3, 2), (4, 2), (2, 8))]
SCHED_SMALL += [("hybrid", 16, 131072, 32, 128, False, 2)]


def build(kind, p, s, h, d, causal, nodes=1):
    if kind == "hybrid":
        return engine.build_hybrid(nodes, p // nodes, s, h, d)
    if kind == "ring":
        return engine.build_ring_attention(p, s, h, d, causal=causal)
    if kind == "token-ring":
        return engine.build_token_ring(p, s, h, d)
    return engine.build_zigzag_token_ring(p, s, h, d)


def schedules():
    out = []
    for args in SCHED_SMALL:
        kind, p, s, h, d, causal = args[:6]
        sc = build(*args)
        tr = engine.trace_from_schedule(sc)
        vol = engine.comm_volume(sc)
        out.append({
            "args": list(args),
            "schedule": canon(sc),
            "ranges": [list(map(list, sc.partition.ranges(r))) for r in range(p)],
            "causal_work": list(partition.causal_work_count(sc.partition)),
            "flops_total": int(sum(c.flops for c in tr.computes)),
            "flops_per_step_rank": [[int(c.step), int(c.rank), int(c.flops)] for c in tr.computes],
            "volume": [[int(st), int(r), kd.value, int(n)] for (st, r, kd), n in sorted(
                vol.entries.items(), key=lambda kv: (kv[0][0], kv[0][1], kv[0][2].value))],
        })
    return out


EXEC_CASES = [
    # name, kind, P, S, H, D, causal, seed, bf16
    ("tr_p2", "token-ring", 2, 64, 2, 16, False, 0, False),
    ("tr_p4", "token-ring", 4, 64, 4, 16, False, 7, False),
    ("zz_p2", "zigzag-token-ring", 2, 32, 2, 8, True, 3, False),
    ("zz_p4", "zigzag-token-ring", 4, 64, 2, 16, True, 1, False),
    ("zz_p8", "zigzag-token-ring", 8, 128, 2, 8, True, 2, False),
    ("ring_causal_p4", "ring", 4, 64, 2, 8, True, 5, False),
    ("ring_p4", "ring", 4, 64, 2, 8, False, 9, False),
    # bf16-rounded inputs at kernel head dims, for the GPU executor fixtures
    ("zz_p4_bf16_d128", "zigzag-token-ring", 4, 1024, 2, 128, True, 31, True),
    ("tr_p2_bf16_d64", "token-ring", 2, 512, 2, 64, False, 32, True),
    ("hy_2x2", "hybrid", 4, 64, 2, 8, False, 12, False, 2),
    ("hy_2x4_bf16_d128", "hybrid", 8, 512, 2, 128, False, 33, True, 2),
    ("hy_3x2_bf16_d64", "hybrid", 6, 768, 2, 64, False, 34, True, 3),
]


def exec_cases():
    arrs, meta = {}, []
    for name, kind, p, s, h, d, causal, seed, bf, *nodes in EXEC_CASES:
        sc = build(kind, p, s, h, d, causal, *nodes)
        q, k, v = rng.attention_inputs(seed, s, h, d)
        if bf:
            q, k, v = to_bf16_f64(q), to_bf16_f64(k), to_bf16_f64(v)
        outs, _ = engine.execute(sc, q, k, v)
        for r in range(p):
            arrs[f"{name}__out{r}"] = outs[r].out
            arrs[f"{name}__lse{r}"] = outs[r].lse
        dense = ringsim.dense_attention_oracle(q, k, v, causal=causal)
        arrs[f"{name}__dense_out"] = dense.out
        arrs[f"{name}__dense_lse"] = dense.lse
        meta.append({"name": name, "args": [kind, p, s, h, d, causal, *nodes], "seed": seed,
                     "bf16": bf})
    return arrs, meta


def cli_volumes():
    """ringsim.cli volume output for the configs shipped in configs/."""
    import io
    from ringsim import cli
    cfg_dir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "configs")
    res = {}
    for name in sorted(os.listdir(cfg_dir)):
        buf = io.StringIO()
        cli.cmd_volume(cli.load_config(os.path.join(cfg_dir, name)), out=buf)
        res[name] = buf.getvalue()
    return res


def main():
    with open(os.path.join(OUT, "cli_volume.json"), "w") as f:
        json.dump(cli_volumes(), f, indent=1)
    with open(os.path.join(OUT, "rng_kats.json"), "w") as f:
        json.dump(rng_kats(), f, indent=1)
    arrs, meta = kernel_cases()
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **arrs)
    with open(os.path.join(OUT, "kernels.json"), "w") as f:
        json.dump(meta, f, indent=1)
    arrs, names = merge_cases()
    np.savez_compressed(os.path.join(OUT, "merge.npz"), **arrs)
    with open(os.path.join(OUT, "merge.json"), "w") as f:
        json.dump(names, f)
    with open(os.path.join(OUT, "schedules.json"), "w") as f:
        json.dump(schedules(), f, separators=(",", ":"))
    arrs, meta = exec_cases()
    np.savez_compressed(os.path.join(OUT, "execute.npz"), **arrs)
    with open(os.path.join(OUT, "execute.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("golden fixtures written to", os.path.abspath(OUT), "backend", ringsim.KERNEL_BACKEND)


if __name__ == "__main__":
    main()
