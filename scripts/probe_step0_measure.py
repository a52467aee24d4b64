"""Per-rank launch times of steps 0 and 1 as cli.measure records them
(zigzag TokenRing, P=8, H=32, D=128, causal), to see whether the slow step 0
of the emulated sweep is every rank or only the first launch after the
host's head-start sleep.  Diagnostic only.

    python scripts/probe_step0_measure.py [S]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20501_b200 import cli  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    cfg = cli.RunConfig.from_dict({
        "problem": {"seq_len": S, "heads": 32, "head_dim": 128, "causal": True, "seed": 0},
        "parallel": {"ranks": 8, "nodes": 1}, "schedule": {"kind": "zigzag-token-ring"}})
    sched, _, _, compute = cli.measure(cfg, repeats=3)
    for st in range(sched.n_steps):
        print(f"step {st}: " + " ".join(f"{t * 1e6:7.1f}" for t in compute[st]) + "  us per rank")


if __name__ == "__main__":
    main()
