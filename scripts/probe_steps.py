"""Per-step launch efficiency of the P-rank schedules on one B200 (diagnostic,
not the bench): every rank's step launch is measured by ``cli.measure`` (CUDA
events around each rank's ComputePlans, ranks run one after another on the
GPU); for each step the TFLOP/s of the slowest rank's launch is printed next
to the launch geometry (pair tiles, waves of 74 CTA pairs).

    python scripts/probe_steps.py [S ...]      (default 32768 65536 131072; P=8, H=32, D=128)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _ablib import maybe_use_env_library  # noqa: E402
maybe_use_env_library()

from paper_2412_20501_b200 import cli, engine  # noqa: E402


def main():
    seqs = [int(x) for x in sys.argv[1:]] or [32768, 65536, 131072]
    P, H, D = 8, 32, 128
    for causal, kind in ((True, "zigzag-token-ring"), (False, "token-ring")):
        for S in seqs:
            cfg = cli.RunConfig.from_dict({
                "problem": {"seq_len": S, "heads": H, "head_dim": D, "causal": causal, "seed": 0},
                "parallel": {"ranks": P, "nodes": 1},
                "schedule": {"kind": kind}})
            sched, _, _, compute = cli.measure(cfg, repeats=3)
            tr = engine.trace_from_schedule(sched)
            flops = [[0.0] * P for _ in range(sched.n_steps)]
            for c in tr.computes:
                flops[c.step][c.rank] += c.flops
            tot_f = tot_t = 0.0
            rows = []
            for st in range(sched.n_steps):
                t = max(compute[st])
                f = max(flops[st])
                if t <= 0 or f <= 0:
                    continue
                tot_f += sum(flops[st])
                tot_t += t
                rows.append(f"{st}:{f / t / 1e12:6.0f}")
            print(f"{kind:18s} S={S:7d} P={P}: per-step TF of the slowest rank  {' '.join(rows)}"
                  f"  | all steps {tot_f / P / tot_t / 1e12:6.0f} TF per GPU")
            sys.stdout.flush()


if __name__ == "__main__":
    main()
