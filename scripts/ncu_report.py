"""Summarise an ncu --set full report of one kernel: key throughput metrics,
stall reasons of the hottest loop, top instructions by stall samples.

    python scripts/ncu_report.py gpurun_out/attn_v2.ncu-rep [--top 25]
"""
import argparse
import csv
import subprocess
from collections import Counter, defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "sm__cycles_elapsed.avg"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    r = list(csv.reader(run([a.rep, "--page", "raw", "--csv"]).splitlines()))
    h, u, v = r[0], r[1], r[2]
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"{k:80s} {v[i]} {u[i]}")
    rows = list(csv.reader(run([a.rep, "--page", "source", "--csv", "--print-source", "sass"])
                           .splitlines()))
    hdr = rows[1]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    cols = [i for i, x in enumerate(hdr) if x.startswith("stall_") and "Not Issued" not in x]
    data = []
    for row in rows[2:]:
        try:
            data.append((int(row[si]), row[1].strip(), int(row[ie]), row))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    by_count = defaultdict(int)
    for s, _, n, _ in data:
        by_count[n] += s
    print("\nstall samples by execution count (loop bodies):")
    for n, s in sorted(by_count.items(), key=lambda x: -x[1])[:6]:
        ops = Counter()
        reasons = Counter()
        for s2, src, n2, row in data:
            if n2 == n:
                op = [o for o in src.split() if not o.startswith("@")][0].split(".")[0]
                ops[op] += 1
                for i in cols:
                    try:
                        reasons[hdr[i]] += int(row[i])
                    except ValueError:
                        pass
        rs = sum(reasons.values()) or 1
        print(f"  exec={n:>12d} samples={100 * s / tot:5.1f}%  instrs={sum(ops.values())}")
        print("    ops:", ", ".join(f"{k}:{c}" for k, c in ops.most_common(14)))
        print("    stalls:", ", ".join(f"{k[6:]}:{100 * c / rs:.0f}%" for k, c in reasons.most_common(6)))
    print(f"\ntop {a.top} instructions by samples:")
    for s, src, n, _ in sorted(data, key=lambda x: -x[0])[:a.top]:
        print(f"  {100 * s / tot:5.1f}% {n:>12d}  {src[:90]}")


if __name__ == "__main__":
    main()
