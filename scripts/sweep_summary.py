"""Markdown tables of a config-4 sweep (the `cli compare` CSVs that
scripts/sweep_config4.sh writes): forward ms (job TFLOP/s) per sequence
length, ring vs TokenRing, at every P -- step-synchronous (every step waits
for the slowest rank's launch) and, where the CSV has them, chained (each
rank's step launches back to back as programmatic dependents, as the runner
issues them).

    python scripts/sweep_summary.py DIR          (reads DIR/compare_{causal,noncausal}_p{2,4,8}.csv)
"""
import csv
import os
import sys


def load(path, chained=False):
    rows = {}
    with open(path) as f:
        for r in csv.DictReader(f):
            if chained:
                if not r.get("chained_total_ms"):
                    continue
                val = (float(r["chained_total_ms"]), float(r["chained_tflops"]))
            else:
                val = (float(r["total_ms"]), float(r["tflops"]))
            rows[(int(r["param_value"]), r["schedule"])] = val
    return rows


def table(d, mode, pair, chained=False):
    ring, tok = pair
    ps = [p for p in (2, 4, 8) if os.path.exists(os.path.join(d, f"compare_{mode}_p{p}.csv"))]
    data = {p: load(os.path.join(d, f"compare_{mode}_p{p}.csv"), chained) for p in ps}
    seqs = sorted({s for p in ps for s, _ in data[p]})
    head = ["S"] + [x for p in ps for x in (f"P={p} {ring}", f"P={p} {tok}", "speed-up")]
    out = ["| " + " | ".join(head) + " |", "|" + "---|" * len(head)]
    for s in seqs:
        cells = [f"{s // 1024}K"]
        for p in ps:
            a, b = data[p].get((s, ring)), data[p].get((s, tok))
            cells += [f"{a[0]:.2f} ({a[1]:.0f})" if a else "-", f"{b[0]:.2f} ({b[1]:.0f})" if b else "-",
                      f"{a[0] / b[0]:.2f}x" if a and b else "-"]
        out.append("| " + " | ".join(cells) + " |")
    return "\n".join(out)


def main():
    d = sys.argv[1]
    for chained in (False, True):
        tag = " (chained step launches)" if chained else " (step-synchronous)"
        print(f"## causal: ring vs zigzag-token-ring{tag}\n")
        print(table(d, "causal", ("ring", "zigzag-token-ring"), chained))
        print(f"\n## noncausal: ring vs token-ring{tag}\n")
        print(table(d, "noncausal", ("ring", "token-ring"), chained))
        print()


if __name__ == "__main__":
    main()
