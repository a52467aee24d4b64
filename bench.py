"""Benchmark of the TokenRing attention path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--seq S] [--impl reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json configs[2], the metric's own config): zigzag
TokenRing forward, S=131072 tokens, 32 heads, d=128, causal, bf16, over N
ranks (strong scaling: the whole sequence is fixed, every rank owns S/N
tokens).  At N=1 the schedule is the reference's trivial single-rank one
(one causal block over the whole sequence, ref engine.py:176-184).

A step = one full TokenRing forward (all P steps + final phase).  ``value``
is whole-job algorithmic TFLOP/s (4*H*D*S(S+1)/2 per step, ref
engine.py:170-173) over the max-over-ranks device time with inputs resident
in HBM; ``e2e`` repeats the measurement through the same public API with the
inputs copied from pinned host memory and the output copied back inside the
timed region.  Every q/k/v tensor is 1 GiB (> 126 MB L2), so no explicit L2
flush is needed between steps.

``--impl reference`` times the reference's own CPU path -- its
``engine.execute`` on the numpy backend (the faster one at scale, BASELINE.md
section 3), from the unmodified install in baseline/_ref, or the oracle port
when that is absent -- on all host cores, one head per process, on a bounded
sample of the same schedule (S=16384, 8 simulated ranks), extrapolated to
the full workload, and prints the same JSON line with "impl": "reference"
(plus the reference's Cython kernels on causal row windows beside it).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("Attention TFLOP/s + tokens/s at 128K seq on 1/2/4/8 B200; exposed comm ms/step")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seq", type=int, default=131072)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--schedule", default="token-ring", choices=["token-ring", "ring"],
                    help="token-ring (default: zigzag TokenRing when causal, the metric's "
                         "workload) or ring (Ring Attention KV rotation, ref engine.py:203-230: "
                         "the config-4 baseline)")
    ap.add_argument("--non-causal", action="store_true",
                    help="non-causal attention (config-4 sweep; TokenRing then uses the "
                         "contiguous partition)")
    ap.add_argument("--trace-out", default=None, metavar="PREFIX",
                    help="after the timed steps, one more forward with every rank's lanes "
                         "measured: PREFIX.json (Chrome trace, the reference's schema), PREFIX.csv "
                         "(the reference's step CSV), PREFIX_exchange.json")
    ap.add_argument("--graph", dest="graph", action="store_true", default=None,
                    help="time CUDA-graph replays of the forward (TokenRingAttention.capture); "
                         "default on for N>1 with the ipc/fused transports")
    ap.add_argument("--no-graph", dest="graph", action="store_false")
    ap.add_argument("--transport", default="fused", choices=["nccl", "ipc", "fused"],
                    help="N>1 exchange: fused (default: Q by copy engines into the peer's "
                         "IPC-mapped buffer, OUT rows stored by the attention epilogue straight "
                         "into the home rank's receive slot), ipc (copy engines both ways) or "
                         "nccl (torch.distributed P2P, the baseline)")
    ap.add_argument("--no-overlap-steps", dest="overlap_steps", action="store_false",
                    help="N>1 ipc/fused: plain stream-ordered step launches instead of "
                         "programmatic dependent launches of the previous step (A/B)")
    return ap.parse_args()


def causal_flops(S, H, D):
    return 4 * H * D * (S * (S + 1) // 2)


def workload_flops(a):
    return 4 * a.heads * a.head_dim * a.seq * a.seq if a.non_causal else \
        causal_flops(a.seq, a.heads, a.head_dim)


def schedule_name(a, n):
    if a.schedule == "ring":
        name = "ring (Ring Attention, KV rotation)"
    else:
        name = "token-ring" if a.non_causal else "zigzag-token-ring"
    return name if n > 1 else name + " (P=1 trivial)"


def workload_config(a, n):
    mask = "non-causal" if a.non_causal else "causal"
    label = "Ring Attention" if a.schedule == "ring" else (
        "TokenRing" if a.non_causal else "zigzag TokenRing")
    return {"workload": f"{label} fwd, S={a.seq}, H={a.heads}, D={a.head_dim}, {mask}, "
                        f"bf16, {n} rank(s)",
            "seq_len": a.seq, "heads": a.heads, "head_dim": a.head_dim, "ranks": n,
            "schedule": schedule_name(a, n), "causal": not a.non_causal,
            "global_batch": 1, "parallelism": f"sp{n}",
            "l2": "inputs larger than L2 (each q/k/v tensor >= 1 GiB at S=131072), no flush"}


# ------------------------------------------------------------------ CPU side
def _cpu_sample_worker(args):
    """One worker: causal row windows of one head (rows at the end of the
    sequence, keys 0..S) through the CPU kernels until ``budget`` seconds of
    work are done.  Returns (algorithmic flops, seconds, rows)."""
    kind, S, D, budget, seed = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    import numpy as np
    rng = np.random.default_rng(seed)
    w = 8 if kind == "reference" else 128          # rows per call (bounded memory)
    k = rng.uniform(-1, 1, (S, 1, D))
    v = rng.uniform(-1, 1, (S, 1, D))
    if kind == "reference":
        from oracle import ref_kernels
        mod = ref_kernels.load()

        def call(q, a0):
            mod.attention_block(q, k, v, 2, a0, 0)
    else:
        from oracle import kernels as ok

        def call(q, a0):
            ok.attention_block(q, k, v, ok.MASK_CAUSAL, a0, 0)
    flops, rows, t0 = 0, 0, time.perf_counter()
    while True:
        a0 = S - w - (rows % (S // 2))
        q = np.ascontiguousarray(rng.uniform(-1, 1, (w, 1, D)))
        call(q, a0)
        flops += 4 * D * (w * a0 + w * (w + 1) // 2)
        rows += w
        dt = time.perf_counter() - t0
        if dt >= budget:
            return flops, dt, rows


def cpu_rate(kind, S, D, budget_s=12.0, workers=None):
    """Aggregate CPU TFLOP/s of the reference kernels on this host: every core
    runs causal row windows of one head -- a bounded sample of the same causal
    workload (per-pair cost is what matters; heads are independent)."""
    import multiprocessing as mpc
    workers = workers or len(os.sched_getaffinity(0))
    ctx = mpc.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(workers) as pool:
        res = pool.map(_cpu_sample_worker, [(kind, S, D, budget_s, 100 + i)
                                            for i in range(workers)])
    wall = time.perf_counter() - t0
    flops = sum(r[0] for r in res)
    busy = max(r[1] for r in res)
    return {"flops": flops, "seconds": busy, "wall": wall, "workers": workers,
            "rows": sum(r[2] for r in res), "tflops": flops / busy / 1e12}


def reference_kind():
    from oracle import ref_kernels
    return "reference" if ref_kernels.load() is not None else "port"


REF_PKG = os.path.join(ROOT, "baseline", "_ref")     # pip --target install of /root/reference
EXEC_SAMPLE_S = 16384                                # sequence of one sampled execute
EXEC_SAMPLE_P = 8                                    # simulated ranks (config 3's schedule)


def _ref_package_ok():
    return os.path.isdir(os.path.join(REF_PKG, "ringsim"))


def _exec_sample_worker(args):
    """One worker: the reference's own executor (``ringsim.engine.execute``,
    ref engine.py:468-638) on its numpy backend (``RINGSIM_KERNELS=python``,
    _kernels_ref.py) over the schedule of the benchmarked workload at H=1,
    S=EXEC_SAMPLE_S, repeated with fresh inputs (one head each -- heads are
    independent) until ``budget`` seconds of execute time.  Without the
    reference install, the oracle port's execute (oracle/schedule.py).
    Returns (algorithmic flops, seconds inside execute, executes)."""
    schedule, causal, S, P, D, budget, seed = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["RINGSIM_KERNELS"] = "python"
    if _ref_package_ok():
        sys.path.insert(0, REF_PKG)
        from ringsim import engine, rng
        if schedule == "ring":
            sched = engine.build_ring_attention(P, S, 1, D, causal=causal)
        elif causal:
            sched = engine.build_zigzag_token_ring(P, S, 1, D)
        else:
            sched = engine.build_token_ring(P, S, 1, D)
        flops = sum(c.flops for c in engine.trace_from_schedule(sched).computes)

        def run(sd):
            q, k, v = rng.attention_inputs(sd, S, 1, D)
            t = time.perf_counter()
            engine.execute(sched, q, k, v)
            return time.perf_counter() - t
    else:
        from oracle import schedule as osch
        from oracle import splitmix
        sched = (osch.ring(P, S, 1, D, causal) if schedule == "ring" else
                 osch.zigzag_token_ring(P, S, 1, D) if causal else osch.token_ring(P, S, 1, D))
        flops = osch.flops(sched, 1, D)

        def run(sd):
            q, k, v = splitmix.attention_inputs(sd, S, 1, D)
            t = time.perf_counter()
            osch.execute(sched, q, k, v)
            return time.perf_counter() - t
    busy, n = 0.0, 0
    while True:
        busy += run(seed + n)
        n += 1
        if busy >= budget:
            return flops * n, busy, n


def host_info():
    """The host facts SURVEY 8(d) asks the CPU baseline to report."""
    return {"os_cpu_count": os.cpu_count(), "affinity_cpus": len(os.sched_getaffinity(0)),
            "openblas_num_threads_per_process": 1}


def cpu_exec_rate(schedule, causal, D, budget_s=8.0, workers=None):
    """Aggregate CPU TFLOP/s of the reference's CPU path on this host: every
    core runs the reference's own ``execute`` of the benchmarked schedule
    (8 simulated ranks, one head per execute) -- a bounded sample of the same
    workload; the numpy backend's rate is flat in S (measured 18.0 / 18.2
    GFLOP/s per core at S=16384 / 32768), so it extrapolates to the full one."""
    import multiprocessing as mpc
    workers = workers or len(os.sched_getaffinity(0))
    ctx = mpc.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(workers) as pool:
        res = pool.map(_exec_sample_worker,
                       [(schedule, causal, EXEC_SAMPLE_S, EXEC_SAMPLE_P, D, budget_s, 1000 + 97 * i)
                        for i in range(workers)])
    wall = time.perf_counter() - t0
    flops = sum(r[0] for r in res)
    busy = max(r[1] for r in res)
    return {"flops": flops, "seconds": busy, "wall": wall, "workers": workers,
            "executes": sum(r[2] for r in res), "tflops": flops / busy / 1e12,
            "kind": "reference" if _ref_package_ok() else "port"}


def _exec_sample_text(r, a):
    what = ("the reference package's own engine.execute (baseline/_ref, RINGSIM_KERNELS=python: "
            "numpy/OpenBLAS, 1 BLAS thread per process)" if r["kind"] == "reference" else
            "the oracle port's execute (oracle/schedule.py, numpy; reference install absent)")
    sched = ("build_ring_attention" if a.schedule == "ring" else
             "build_token_ring" if a.non_causal else "build_zigzag_token_ring")
    return (f"{r['workers']} processes, each running {what} of {sched}({EXEC_SAMPLE_P}, "
            f"{EXEC_SAMPLE_S}, 1, {a.head_dim}) on fresh one-head inputs: {r['executes']} executes "
            f"in {r['seconds']:.1f} s; aggregate throughput extrapolated to the full workload "
            f"(S={a.seq}, H={a.heads})")


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    S, H, D = a.seq, a.heads, a.head_dim
    total = workload_flops(a)
    rates = []
    for i in range(a.warmup + a.steps):
        r = cpu_exec_rate(a.schedule, not a.non_causal, D, budget_s=2.0 if i < a.warmup else 6.0)
        if i >= a.warmup:
            rates.append(r)
    tflops = statistics.median(r["tflops"] for r in rates)
    sec_per_step = total / (tflops * 1e12)
    r0 = rates[0]
    # the reference's other backend (Cython, compiled from its own source by
    # oracle/Makefile) on causal row windows, for comparison
    cy = None
    if reference_kind() == "reference" and not a.non_causal:
        c = cpu_rate("reference", S, D, budget_s=6.0)
        cy = {"value": c["tflops"], "unit": "TFLOP/s", "cores": c["workers"],
              "sample": f"ringsim/_kernels.pyx attention_block on {c['rows']} causal query rows "
                        f"(8-row windows near the end of S={S}), {c['seconds']:.1f} s",
              "faster_backend": "numpy execute" if tflops >= c["tflops"] else "cython kernels"}
    line = {
        "impl": "reference", "metric": METRIC, "value": tflops, "unit": "TFLOP/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": sec_per_step * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SplitMix64 uniform[-1,1) fp64)",
        "config": workload_config(a, a.gpus),
        "tokens_per_s": S / sec_per_step,
        "cpu_baseline": {"value": tflops, "unit": "TFLOP/s", "cores": r0["workers"],
                         "kind": r0["kind"], "path": "engine.execute (numpy backend)",
                         "extrapolated": True, "sample": _exec_sample_text(r0, a),
                         "host": host_info()},
        "cpu_baseline_cython": cy,
        "e2e": {"value": tflops, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU side
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        loaded = [x for x in sm if mx and x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


def ncu_traffic():
    """DRAM bytes per attention launch from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "attn_ncu_summary.json")) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch_128k")
    except Exception:
        return None


def e2e_pipelined(make_runner, q, k, v, steps, barrier, allmax, groups, edge=0,
                  return_outputs=False):
    """End to end through the public API with host buffers.  Heads are
    independent, so the inputs live on the host as head groups (contiguous
    (T, heads, D) pinned buffers) and every step runs one TokenRing forward
    per group (a TokenRingAttention over that many heads): H2D of the next
    group's q/k/v and D2H of the previous group's bf16 output and lse overlap
    the current group's compute on their own streams, so only the first
    group's input copy (pipeline fill) and the last group's output copy
    (drain) are exposed per timed run -- and with ``edge`` > 0 the run's very
    first and very last groups are split so that those two are only ``edge``
    heads each.  Every step's copies are inside the timed region.  Returns ms
    per step (max over ranks); with ``return_outputs`` also the pinned host
    outputs, {(h0, h1): [[out, lse] for the two step parities]}."""
    import torch
    T, H, D = q.shape
    G = groups
    hg = H // G
    edge = edge if 0 < edge < hg else 0
    runners = {}

    def runner_for(n):
        if n not in runners:
            runners[n] = make_runner(n)
        return runners[n]

    cur = torch.cuda.current_stream()
    cs_in, cs_out = torch.cuda.Stream(), torch.cuda.Stream()
    host_in, host_out = {}, {}

    def host_bufs(h0, h1):
        if (h0, h1) not in host_in:
            host_in[(h0, h1)] = [t[:, h0:h1].contiguous().cpu().pin_memory() for t in (q, k, v)]
            host_out[(h0, h1)] = [
                [torch.zeros((T, h1 - h0, D), dtype=torch.bfloat16).pin_memory(),
                 torch.zeros((h1 - h0, T), dtype=torch.float32).pin_memory()] for _ in range(2)]
        return host_in[(h0, h1)], host_out[(h0, h1)]

    # device staging: two slots of flat buffers sized for the largest group,
    # viewed as (T, n, D) for an n-head group
    dev_flat = [[torch.empty(T * hg * D, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
                for _ in range(2)]
    obf_flat = [torch.empty(T * hg * D, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    lsd_flat = [torch.empty(hg * T, dtype=torch.float32, device="cuda") for _ in range(2)]
    ev = {n: [torch.cuda.Event() for _ in range(2)] for n in ("in", "used", "out", "d2h")}

    def pieces(st, g, n):
        h0, h1 = g * hg, (g + 1) * hg
        cuts = [h0, h1]
        if edge and st == 0 and g == 0:
            cuts.insert(1, h0 + edge)
        if edge and st == n - 1 and g == G - 1:
            cuts.insert(len(cuts) - 1, h1 - edge)
        return [(st, a, b) for a, b in zip(cuts[:-1], cuts[1:])]

    def run(n):
        units = [u for st in range(n) for g in range(G) for u in pieces(st, g, n)]
        for _, a, b in units:
            host_bufs(a, b)
            runner_for(b - a)

        def h2d(u):
            sl = u % 2
            _, a, b = units[u]
            with torch.cuda.stream(cs_in):
                if u >= 2:
                    cs_in.wait_event(ev["used"][sl])
                for d, hsrc in zip(dev_flat[sl], host_in[(a, b)]):
                    d[:hsrc.numel()].view(hsrc.shape).copy_(hsrc, non_blocking=True)
                ev["in"][sl].record(cs_in)
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(cur)
        cs_in.wait_stream(cur)
        cs_out.wait_stream(cur)
        h2d(0)
        for u, (st, a, b) in enumerate(units):
            sl = u % 2
            nh = b - a
            if u + 1 < len(units):
                h2d(u + 1)
            cur.wait_event(ev["in"][sl])
            res = runner_for(nh)(*[d[:T * nh * D].view(T, nh, D) for d in dev_flat[sl]])
            ev["used"][sl].record(cur)
            if u >= 2:
                cur.wait_event(ev["d2h"][sl])
            obf = obf_flat[sl][:T * nh * D].view(T, nh, D)
            lsd = lsd_flat[sl][:nh * T].view(nh, T)
            obf.copy_(res.out)                  # bf16 output, the inputs' dtype
            lsd.copy_(res.lse)
            ev["out"][sl].record(cur)
            with torch.cuda.stream(cs_out):
                cs_out.wait_event(ev["out"][sl])
                oh, lh = host_out[(a, b)][st % 2]
                oh.copy_(obf, non_blocking=True)
                lh.copy_(lsd, non_blocking=True)
                ev["d2h"][sl].record(cs_out)
        cur.wait_stream(cs_out)
        end.record(cur)
        return start, end

    run(2)                      # warm-up (allocations, first-touch of pinned pages)
    barrier()
    torch.cuda.synchronize()
    s, e = run(steps)
    torch.cuda.synchronize()
    barrier()
    ms = allmax([s.elapsed_time(e) / steps])[0]
    return (ms, host_out) if return_outputs else ms


def exchange_report(world, runner, xsum, n_fwd, shared):
    """Per-direction exchange of the TokenRing schedule (Q
    forward, OUT_LSE reverse) in GB/s against NVLink 5's 900 GB/s per
    direction.  Bytes are algorithmic (Q: rows*H*D*2, OUT: rows*H*(2D+4)),
    summed over all ranks; time is the device time of the transfers.  The
    Ring-Attention baseline moves KV blocks instead (rows*H*D*2*2 per hop)."""
    if world == 1:
        return None
    q_b, q_ms, o_b, o_ms, k_b, k_ms = xsum
    fwd = max(1, n_fwd)
    rep = {"peak_gbs_per_direction": 900.0,
           "q_bytes_per_forward": q_b / fwd, "out_bytes_per_forward": o_b / fwd,
           "q_gbs": q_b / (q_ms * 1e-3) / 1e9 if q_ms > 0 else None,
           "out_gbs": o_b / (o_ms * 1e-3) / 1e9 if o_ms > 0 else None,
           "transport": runner.transport,
           # ipc / fused: step launches are programmatic dependents of the previous step
           "overlapped_steps": bool(runner.overlap_steps and runner.transport in ("ipc", "fused"))}
    if k_b > 0:
        rep["kv_bytes_per_forward"] = k_b / fwd
        rep["kv_gbs"] = k_b / (k_ms * 1e-3) / 1e9 if k_ms > 0 else None
    if runner.transport == "fused":
        rep["out_path"] = ("epilogue stores into the home's slot; out_gbs = bytes over the "
                           "launch that computes them (link load, not link peak)")
    if runner.transport == "nccl":
        rep["note"] = "NCCL P2P runs on NCCL's streams; only exposed comm is timed"
    if shared:
        rep["note"] = "all ranks share one GPU: copies are device-local, not NVLink"
    return rep


def run_ours(a):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    # TR_BENCH_SHARED_DEVICE=1: test mode for the multi-rank flow on a one-GPU
    # box -- every rank on cuda:0, copy-engine transport, gloo for the host
    # collectives.  Numbers from it are not scaling numbers.
    shared = os.environ.get("TR_BENCH_SHARED_DEVICE") == "1" and world > 1
    if shared and a.transport not in ("ipc", "fused"):
        raise SystemExit("TR_BENCH_SHARED_DEVICE=1 needs --transport ipc or fused")
    dev_index = 0 if shared else local
    torch.cuda.set_device(dev_index)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def allsum(vals):
        if world == 1:
            return list(vals)
        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return [float(x) for x in t.tolist()]

    def allmax(vals):
        if world == 1:
            return list(vals)
        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t.tolist()]

    from paper_2412_20501_b200 import kernels, rng
    from paper_2412_20501_b200.ring import TokenRingAttention

    S, H, D = a.seq, a.heads, a.head_dim
    transport = a.transport
    if world > 1 and not shared and transport in ("ipc", "fused"):
        # peer-memory transports need a P2P path between every pair of GPUs;
        # decide collectively so every rank runs the same transport
        n = torch.cuda.device_count()
        ok = all(torch.cuda.can_device_access_peer(dev_index, d) for d in range(n) if d != dev_index)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if flag.item() == 0:
            print(f"bench: no P2P path between all GPUs; transport {transport} -> nccl",
                  file=sys.stderr)
            transport = "nccl"
    causal = not a.non_causal
    runner = TokenRingAttention(S, H, D, causal=causal, record_timeline=True,
                                transport=transport, schedule=a.schedule,
                                overlap_steps=a.overlap_steps)
    runners = [runner]
    q, k, v = rng.local_inputs(a.seed, runner.part, rank, H, D)
    total_flops = workload_flops(a)

    def barrier():
        if world > 1:
            dist.barrier()

    host_ms = [0.0]

    def timed(fn, steps):
        barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        h0 = time.perf_counter()
        for _ in range(steps):
            fn()
        # host time to enqueue the steps (no sync inside): when it exceeds the
        # device time the GPU waits on the host
        host_ms[0] = (time.perf_counter() - h0) * 1e3 / steps
        e.record()
        torch.cuda.synchronize()
        barrier()
        return allmax([s.elapsed_time(e) / steps])[0]

    timelines = []

    # CUDA-graph replay of the whole forward (TokenRingAttention.capture): one
    # graph launch of host work per step instead of the step loop's launches
    use_graph = a.graph if a.graph is not None else (world > 1 and transport in ("ipc", "fused"))

    def step():
        runner(q, k, v)
        timelines.append(runner.timeline)

    for _ in range(a.warmup):
        step()
    timelines.clear()
    launches_per_step = None
    if use_graph:
        l0 = kernels.LAUNCHES
        runner(q, k, v)                        # one eager forward: count its launches
        launches_per_step = kernels.LAUNCHES - l0
        runner.record_timeline = False
        runner.capture(q, k, v, warmup=1)
        timelines.clear()
    launches0 = kernels.LAUNCHES
    with ClockSampler(dev_index) as clk:
        ms = timed(step, a.steps)
    host_enqueue_ms = allmax([host_ms[0]])[0]
    launches = ((kernels.LAUNCHES - launches0) // a.steps * a.steps if launches_per_step is None
                else launches_per_step * a.steps)
    torch.cuda.synchronize()
    if use_graph:
        # the per-step lanes (exposed comm, kernel time, exchange) from eager
        # forwards with CUDA events, after the timed replays
        timelines.clear()
        runner.record_timeline = True
        for _ in range(2):
            runner._forward(q, k, v)
            timelines.append(runner.timeline)
        torch.cuda.synchronize()

    # exposed comm (stall of the compute stream on comm events) and the
    # attention kernel's own device time, from the per-step CUDA events
    stall, kern_ms, kern_flops, nlaunch = 0.0, 0.0, 0, 0
    for tl in timelines:
        for ev in tl:
            stall += ev["start"].elapsed_time(ev["comm_ready"])
            if "grant_wait" in ev:             # fused: wait for the home's slot grant
                stall += ev["grant_wait"].elapsed_time(ev["granted"])
            if "attn_start" in ev:
                kern_ms += ev["attn_start"].elapsed_time(ev["attn_end"])
                kern_flops += ev["attn_flops"]
                nlaunch += 1
    # exchange: copy-engine transfers timed on the copy stream (ipc: Q and
    # OUT; fused: Q, while OUT rides inside the attention launch that
    # computes it, so its rate is the bytes over that launch's time)
    xq_b = xq_ms = xo_b = xo_ms = xk_b = xk_ms = 0.0
    for tl in timelines:
        for ev in tl:
            for e0, e1, nb in ev.get("q_copies", ()):
                xq_b += nb
                xq_ms += e0.elapsed_time(e1)
            for e0, e1, nb in ev.get("kv_copies", ()):   # ring / hybrid: KV rotation
                xk_b += nb
                xk_ms += e0.elapsed_time(e1)
            for e0, e1, nb in ev.get("o_copies", ()):
                xo_b += nb
                xo_ms += e0.elapsed_time(e1)
            if "o_push_bytes" in ev:
                xo_b += ev["o_push_bytes"]
                xo_ms += ev["attn_start"].elapsed_time(ev["attn_end"])
    xsum = allsum([xq_b, xq_ms, xo_b, xo_ms, xk_b, xk_ms])
    exposed = stall / max(1, len(timelines))
    attn_avg_ms = kern_ms / max(1, nlaunch)
    attn_flops_per_launch = kern_flops / max(1, nlaunch)
    exposed, attn_avg_ms = allmax([exposed, attn_avg_ms])

    if a.trace_out:
        from paper_2412_20501_b200 import timeline as tl_mod
        barrier()
        torch.cuda.synchronize()
        origin = torch.cuda.Event(enable_timing=True)
        origin.record()
        runner._forward(q, k, v)           # eager, with its per-stream events
        torch.cuda.synchronize()
        recs = tl_mod.rank_records(runner, origin)
        if world > 1:
            everyone = [None] * world
            dist.all_gather_object(everyone, recs)
        else:
            everyone = [recs]
        if rank == 0:
            records = dict(enumerate(everyone))
            os.makedirs(os.path.dirname(os.path.abspath(a.trace_out)), exist_ok=True)
            with open(a.trace_out + ".json", "w") as f:
                f.write(tl_mod.emit_chrome_trace(records))
            with open(a.trace_out + ".csv", "w") as f:
                f.write(tl_mod.summary_csv(records, runner.sched.kind, world, S, H, D))
            with open(a.trace_out + "_exchange.json", "w") as f:
                json.dump(dict(tl_mod.exchange_summary(records), transport=runner.transport,
                               shared_device=shared, schedule=runner.sched.kind), f, indent=1)

    # end-to-end through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        e2e_steps = max(2, a.steps)     # pipeline fill/drain amortised over the K steps
        # head groups: as many as keep each step launch >= ~7 waves of CTAs
        # (256-row q tiles x heads, one CTA per SM), at most TR_BENCH_MAX_GROUPS
        ctas_per_head = S // (256 * world)
        max_g = int(os.environ.get("TR_BENCH_MAX_GROUPS", "4"))
        groups = next(g for g in (8, 4, 2, 1)
                      if g <= max_g and H % g == 0
                      and (g == 1 or ctas_per_head * (H // g) >= 7 * 148))
        def make_runner(hg):
            runners.append(TokenRingAttention(S, hg, D, causal=causal, transport=transport,
                                              schedule=a.schedule, overlap_steps=a.overlap_steps))
            return runners[-1]
        # the run's first and last groups split off a quarter-size piece, so the
        # exposed pipeline fill / drain is a quarter of a group's copy
        edge = (H // groups) // 4
        e2e_ms = e2e_pipelined(make_runner, q, k, v, e2e_steps, barrier, allmax, groups, edge)
        h2d = 3 * q.numel() * 2 * world
        d2h = (q.numel() * 2 + runner.acc_lse.numel() * 4) * world
        e2e = {"value": total_flops / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
               "steps": e2e_steps, "head_groups": groups, "edge_heads": edge,
               "api": "TokenRingAttention.__call__ -> tr_attention_segments(_push) / tr_merge_n "
                      "(C ABI), one call per head group of H/head_groups heads; each step's "
                      "q/k/v copied in from pinned host memory and its bf16 output + lse "
                      "copied out, group by group, on copy streams double-buffered against "
                      "the neighbouring groups' compute (the run's first and last groups split "
                      "off edge_heads-head pieces to shorten the exposed fill and drain)"}

    if rank == 0:
        peaks, peak_src = measured_peaks()
        peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        achieved = attn_flops_per_launch / (attn_avg_ms * 1e-3) / 1e12 if attn_avg_ms > 0 else 0.0
        line = {
            "metric": METRIC, "value": total_flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": f"synthetic (SplitMix64 uniform[-1,1) -> bf16, seed {a.seed}, generated on "
                    "device per rank shard)",
            "config": dict(workload_config(a, world),
                           transport=runner.transport if world > 1 else "none (1 rank)",
                           **({"test_mode": "all ranks share cuda:0 (TR_BENCH_SHARED_DEVICE)"}
                              if shared else {})),
            "tokens_per_s": S / (ms * 1e-3),
            "exposed_comm_ms_per_step": exposed,
            "host_enqueue_ms_per_step": host_enqueue_ms,
            "cuda_graph": bool(use_graph),
            "exchange": exchange_report(world, runner, xsum, len(timelines), shared),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": ncu_traffic(),
                         "kernel": "tr::attn_fwd_pair2_kernel (CTA pairs, cta_group::2)",
                         "flops_per_launch": attn_flops_per_launch,
                         "avg_launch_ms": attn_avg_ms,
                         "peak_kind": f"bf16_tflops_sustained ({peak_src})",
                         "frac_of_burst": achieved / peaks["bf16_tflops"],
                         "frac_of_spec_2250": achieved / 2250.0},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if not a.no_cpu_baseline:
            r = cpu_exec_rate(a.schedule, causal, D, budget_s=10.0)
            line["cpu_baseline"] = {
                "value": r["tflops"], "unit": "TFLOP/s", "cores": r["workers"], "kind": r["kind"],
                "path": "engine.execute (numpy backend)", "extrapolated": True,
                "sample": _exec_sample_text(r, a), "host": host_info()}
        print(json.dumps(line), flush=True)
    if world > 1:
        for r in runners:
            if hasattr(r, "peer"):
                r.close()
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
