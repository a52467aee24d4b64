"""Measured-lane export (paper_2412_20501_b200.timeline) on synthetic event
records: the reference's Chrome-trace schema (netsim.py:277-304) and step CSV
(cli.py:243-255), exposed comm and per-direction rates; and the runner
records real lanes over gloo (CPU, oracle ops with fake events)."""

import json

from paper_2412_20501_b200 import timeline


class Ev:
    def __init__(self, t):
        self.t = t

    def elapsed_time(self, other):
        return other.t - self.t


def _runner(events):
    class R:
        timeline = events
    return R


def test_rank_records_and_exports():
    E = Ev
    tl0 = [{"start": E(0.0), "comm_ready": E(0.0), "attn_start": E(0.1), "attn_end": E(1.6),
            "computed": E(1.6), "attn_flops": 10,
            "q_copies": [(E(0.1), E(0.4), 3_000_000)]},
           {"start": E(1.6), "comm_ready": E(1.7), "attn_start": E(1.7), "attn_end": E(3.2),
            "computed": E(3.3), "o_push_bytes": 4_000_000},
           {"start": E(3.3), "comm_ready": E(3.5)}]                  # fused: final fold wait
    recs = timeline.rank_records(_runner(tl0), E(0.0))
    assert [r["step"] for r in recs] == [0, 1, 2]
    assert recs[0]["compute"] == (0.1, 1.6) and recs[0]["send"] == (0.1, 0.4)
    assert recs[1]["send"] == (1.7, 3.2) and recs[1]["rev_bytes"] == 4_000_000
    assert recs[2]["final"] and "compute" not in recs[2]
    records = {0: recs, 1: recs}
    ev = json.loads(timeline.emit_chrome_trace(records))
    assert all(set(e) == {"name", "ph", "ts", "dur", "pid", "tid"} for e in ev)
    assert {e["tid"] for e in ev} == {"compute", "send", "recv"}
    assert ev == sorted(ev, key=lambda e: (e["pid"], e["ts"], ("compute", "send", "recv").index(e["tid"])))
    first = [e for e in ev if e["pid"] == 0 and e["name"] == "step0"]
    assert {(e["tid"], e["ts"], e["dur"]) for e in first} == {("compute", 100, 1500), ("send", 100, 300)}
    csv = timeline.summary_csv(records, "zigzag-token-ring", 2, 64, 2, 8).splitlines()
    assert csv[0] == timeline.SUMMARY_HEADER
    assert csv[1].startswith("zigzag-token-ring,2,64,2,8,0,1.500000,0.300000,0.000000,1.600000")
    assert csv[-1] == "zigzag-token-ring,2,64,2,8,total,,,,3.500000"
    x = timeline.exchange_summary(records)
    assert abs(x["exposed_comm_ms_per_forward"] - 0.3) < 1e-9
    assert abs(x["forward_gbs"] - 3e6 / 0.3e-3 / 1e9) < 1e-6
