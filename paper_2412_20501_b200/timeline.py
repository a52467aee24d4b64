"""Measured step timeline of the multi-process runner, in the reference's
trace formats.

The reference draws its timeline from a model: ``netsim.simulate``
(netsim.py:216-274) turns the schedule's messages into per-step compute /
send / recv durations on an analytic topology, ``emit_chrome_trace``
(netsim.py:277-304) renders them as Trace Event JSON (pid = rank, tid in
{compute, send, recv}) and ``summary_csv`` (cli.py:243-255) as one row per
step.  Here every lane is MEASURED with CUDA events the runner records on its
own streams (``TokenRingAttention(record_timeline=True)``):

* compute -- the step's attention launch on the compute stream;
* send    -- this rank's outgoing transfers of the step: copy-engine copies
  of Q / KV (forward) and OUT_LSE (reverse, ``ipc``) on the copy stream; with
  the ``fused`` transport the OUT rows leave inside the attention launch, so
  the reverse send lane is that launch;
* recv    -- how long the compute stream waited for the step's inbound
  messages (flag waits / NCCL completion), i.e. the EXPOSED part of the
  exchange.

Times are milliseconds from each rank's origin event, recorded right after a
barrier, so ranks line up to within the barrier's skew.
"""

from __future__ import annotations

import json
import math

LANES = ("compute", "send", "recv")
SUMMARY_HEADER = "schedule,ranks,seq_len,heads,head_dim,step,compute_ms,send_ms,recv_ms,step_ms"


def rank_records(runner, origin) -> list:
    """Per-step lane intervals of this rank's last forward (``runner.timeline``),
    in ms since ``origin`` (a CUDA event recorded before the forward, after a
    barrier).  Call after the device has synchronised."""
    def t(ev):
        return origin.elapsed_time(ev)

    recs = []
    for i, ev in enumerate(runner.timeline):
        if "start" not in ev:
            continue
        rec = {"step": i, "start": t(ev["start"]),
               "ready": t(ev["comm_ready"]) if "comm_ready" in ev else t(ev["start"]),
               "end": t(ev["computed"]) if "computed" in ev else
               (t(ev["comm_ready"]) if "comm_ready" in ev else t(ev["start"])),
               "final": "computed" not in ev}
        if "attn_start" in ev:
            rec["compute"] = (t(ev["attn_start"]), t(ev["attn_end"]))
            rec["flops"] = ev.get("attn_flops", 0)
        fwd, rev = [], []
        fb = rb = 0
        for key, bucket in (("q_copies", fwd), ("kv_copies", fwd), ("o_copies", rev)):
            for e0, e1, nb in ev.get(key, ()):
                bucket.append((t(e0), t(e1)))
                if bucket is fwd:
                    fb += nb
                else:
                    rb += nb
        if "o_push_bytes" in ev and "compute" in rec:
            rev.append(rec["compute"])          # fused: OUT rides the attention launch
            rb += ev["o_push_bytes"]
        spans = fwd + rev
        if spans:
            rec["send"] = (min(a for a, _ in spans), max(b for _, b in spans))
        rec["fwd_bytes"], rec["rev_bytes"] = fb, rb
        rec["fwd_ms"] = sum(b - a for a, b in fwd)
        rec["rev_ms"] = sum(b - a for a, b in rev)
        rec["recv"] = (rec["start"], rec["ready"])
        recs.append(rec)
    return recs


def emit_chrome_trace(records: dict) -> str:
    """{rank: rank_records(...)} -> Trace Event Format JSON in the reference's
    schema (netsim.py:277-304): one complete ('X') event per rank, step and
    nonzero lane, name 'step<i>', integer microseconds (floored), pid = rank,
    tid = lane, ordered by (pid, ts, lane) -- with measured start times."""
    order = {lane: i for i, lane in enumerate(LANES)}
    events = []
    for rank in sorted(records):
        for rec in records[rank]:
            for lane in LANES:
                if lane not in rec:
                    continue
                a, b = rec[lane]
                dur = math.floor((b - a) * 1e3)
                if dur <= 0:
                    continue
                events.append({"name": f"step{rec['step']}", "ph": "X",
                               "ts": math.floor(a * 1e3), "dur": dur, "pid": rank, "tid": lane})
    events.sort(key=lambda e: (e["pid"], e["ts"], order[e["tid"]]))
    return json.dumps(events, separators=(",", ":"))


def step_rows(records: dict) -> list:
    """Per step: max over ranks of each lane's duration and of the step span
    (ms), the reference's step-synchronous summary (cli.py:243-255)."""
    steps = sorted({rec["step"] for recs in records.values() for rec in recs})
    rows = []
    for st in steps:
        per = [rec for recs in records.values() for rec in recs if rec["step"] == st]
        dur = {lane: max((rec[lane][1] - rec[lane][0]) if lane in rec else 0.0 for rec in per)
               for lane in LANES}
        rows.append((st, dur["compute"], dur["send"], dur["recv"],
                     max(rec["end"] - rec["start"] for rec in per)))
    return rows


def summary_csv(records: dict, kind: str, ranks: int, seq_len: int, heads: int,
                head_dim: int) -> str:
    """The reference's step CSV (``SUMMARY_HEADER``, cli.py:27, 243-255) from
    measured lanes; the total row is the forward's span (max over ranks)."""
    prefix = f"{kind},{ranks},{seq_len},{heads},{head_dim}"
    lines = [SUMMARY_HEADER]
    for st, c, s_, r_, span in step_rows(records):
        lines.append(f"{prefix},{st},{c:.6f},{s_:.6f},{r_:.6f},{span:.6f}")
    lines.append(f"{prefix},total,,,,{forward_ms(records):.6f}")
    return "\n".join(lines) + "\n"


def forward_ms(records: dict) -> float:
    return max(max(rec["end"] for rec in recs) - min(rec["start"] for rec in recs)
               for recs in records.values() if recs)


def exchange_summary(records: dict, link_gbs: float = 900.0) -> dict:
    """Exposed comm per step (compute-stream waits), and per direction the
    algorithmic bytes and the rate over the transfers' own device time."""
    n_steps = max(1, max(len(recs) for recs in records.values()))
    waits = [sum(rec["ready"] - rec["start"] for rec in recs) for recs in records.values()]
    fb = sum(rec["fwd_bytes"] for recs in records.values() for rec in recs)
    rb = sum(rec["rev_bytes"] for recs in records.values() for rec in recs)
    fms = sum(rec["fwd_ms"] for recs in records.values() for rec in recs)
    rms = sum(rec["rev_ms"] for recs in records.values() for rec in recs)
    return {"forward_ms": forward_ms(records),
            "exposed_comm_ms_per_step": max(waits) / n_steps,
            "exposed_comm_ms_per_forward": max(waits),
            "forward_bytes": fb, "reverse_bytes": rb,
            "forward_gbs": fb / (fms * 1e-3) / 1e9 if fms > 0 else None,
            "reverse_gbs": rb / (rms * 1e-3) / 1e9 if rms > 0 else None,
            "link_gbs_per_direction": link_gbs}
