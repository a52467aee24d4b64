"""One rank's TokenRing forward compute lane on one B200, with and without
programmatic dependent launch between its step launches (diagnostic, not the
bench).

Each GPU of a P-rank run executes exactly its own rank's step launches one
after another; with the exchange hidden (the measured lanes show the Q for
step s+1 landed long before step s ends) that chain IS the rank's forward.
Here rank r's step launches of the real schedule run back to back on one
stream, each into its own output buffer:

  plain    -- stream-ordered launches (a step's grid starts after the whole
              previous grid; its last partial wave idles the other SMs)
  overlap  -- steps >= 1 as programmatic dependents (tr_set_launch_overlap):
              their CTAs take the SMs the previous step's last wave frees

Prints per shape the chain time of the slowest rank for both, the gain, and
whether the outputs are bit-identical.

    python scripts/probe_pdl.py [S ...]      (default 32768 65536 131072; P=8, H=32, D=128)
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2412_20501_b200 import engine, kernels, rng  # noqa: E402


def rank_steps(sched, r):
    ch = sched.chunks
    steps = []
    for plan in sched.steps:
        cps = plan.computes[r]
        if not cps:
            continue
        qs, ks, _ = engine.group_computes(sched, cps)
        steps.append(([(ch[a].start, ch[a].tokens, ch[a].start) for a in qs],
                      [(ch[b].start, ch[b].tokens, ch[b].start) for b in ks],
                      sum(engine.compute_flops(cp.mask, ch[cp.q_chunk].tokens,
                                               ch[cp.kv_chunk].tokens, sched.heads,
                                               sched.head_dim) for cp in cps)))
    return steps


MODES = ("plain", "overlap", "overlap+event", "overlap+flagwait", "overlap+event+flagwait")


def run_chain(q, k, v, steps, outs, causal, mode, flag):
    overlap = mode != "plain"
    for i, (qs, ks, _) in enumerate(steps):
        o, l = outs[i]
        with kernels.overlap_launches(after_prev=overlap and i > 0, release_next=overlap):
            if i > 0 and "event" in mode:        # what the runner records between steps
                torch.cuda.Event().record()
            if i > 0 and "flagwait" in mode:     # an already satisfied message wait
                kernels.flag_wait_(flag, 1)
            kernels.attention_segments(q, k, v, qs, ks, causal, o, l)


def main():
    seqs = [int(x) for x in sys.argv[1:]] or [32768, 65536, 131072]
    P, H, D, reps = 8, 32, 128, 7
    torch.cuda.set_device(0)
    for causal, build in ((True, engine.build_zigzag_token_ring), (False, engine.build_token_ring)):
        for S in seqs:
            sched = build(P, S, H, D)
            q, k, v = rng.attention_inputs(0, S, H, D)
            res = {m: [] for m in MODES}
            flag = torch.ones(1, dtype=torch.int64, device=q.device)
            same = True
            flops_max = 0
            for r in range(P):
                steps = rank_steps(sched, r)
                flops_max = max(flops_max, sum(f for _, _, f in steps))
                outs = {m: [(torch.empty_like(q), torch.empty((H, S), device=q.device))
                             for _ in steps] for m in ("plain", "overlap")}
                times = {m: [] for m in MODES}
                for it in range(reps + 1):
                    for m in MODES:
                        torch.cuda.synchronize()
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record()
                        run_chain(q, k, v, steps, outs["plain" if m == "plain" else "overlap"],
                                  causal, m, flag)
                        e1.record()
                        torch.cuda.synchronize()
                        if it > 0:
                            times[m].append(e0.elapsed_time(e1))
                for (qs, _, _), (oa, la), (ob, lb) in zip(steps, outs["plain"], outs["overlap"]):
                    for r0, n, _ in qs:
                        same &= torch.equal(oa[r0:r0 + n], ob[r0:r0 + n])
                        same &= torch.equal(la[:, r0:r0 + n], lb[:, r0:r0 + n])
                for m in MODES:
                    res[m].append(statistics.median(times[m]))
            a = max(res["plain"])
            cols = "  ".join(f"{m} {max(res[m]):.3f} ms ({flops_max / max(res[m]) / 1e9:.0f} TF, "
                             f"{100 * (a / max(res[m]) - 1):+.1f} %)" for m in MODES)
            print(f"{sched.kind:18s} S={S:7d} P={P}: slowest rank chain: {cols}  "
                  f"bit-identical {same}")
            sys.stdout.flush()
            del q, k, v


if __name__ == "__main__":
    main()
