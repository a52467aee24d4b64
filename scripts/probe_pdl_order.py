"""Stream-order semantics around a programmatic dependent launch (diagnostic).

On one stream: A = a long attention launch (plain), then B = a short
attention launch as a programmatic dependent of A (it may run while A's last
wave still runs), then C = a plain tiny launch.  Events: eA after A, eB after
B.  The runner relies on two orderings, checked here on the device:

  1. an event recorded after B completes only once A has completed too
     (elapsed_time(eA, eB) >= 0; host polling never sees eB done, eA not);
  2. a plain launch after B starts only after A completed (C's output is the
     sum A wrote: C reads A's out).

    python scripts/probe_pdl_order.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2412_20501_b200 import kernels, rng  # noqa: E402


def main():
    torch.cuda.set_device(0)
    D = 128
    # A: 75 pair tiles of 256 kv tiles each (15 heads x 5 x 512 rows vs 32K
    # keys, non-causal): a full first wave of 74 CTA pairs, then ONE pair
    # alone for a whole item -- B (a programmatic dependent) runs on the idle
    # SMs during that lone item and finishes long before A
    HA, TA, TK = 15, 2560, 32768
    q, k, v = rng.attention_inputs(1, TK, HA, D)
    qa = q[:TA].contiguous()
    outA = torch.empty_like(qa)
    lseA = torch.empty((HA, TA), device=q.device)
    qs, ks, vs = q[:512].contiguous(), k[:512].contiguous(), v[:512].contiguous()
    outB = torch.empty_like(qs)
    lseB = torch.empty((HA, 512), device=q.device)
    bad_events = bad_host = bad_read = 0
    trials = 10

    def chain(with_b, overlap):
        with kernels.overlap_launches(after_prev=False, release_next=overlap):
            kernels.attention_block(qa, k, v, kernels.MASK_NONE, out=outA, lse=lseA)   # A
        eA.record()
        if with_b:
            with kernels.overlap_launches(after_prev=overlap):
                kernels.attention_block(qs, ks, vs, kernels.MASK_NONE, out=outB, lse=lseB)  # B
        eB.record()

    for t in range(trials):
        times = {}
        for mode in ("A only", "A+B plain", "A+B overlap"):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            eA = torch.cuda.Event(enable_timing=True)
            eB = torch.cuda.Event(enable_timing=True)
            e0.record()
            chain(mode != "A only", mode == "A+B overlap")
            torch.cuda.synchronize()
            times[mode] = e0.elapsed_time(eB)
        outA.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        eA = torch.cuda.Event(enable_timing=True)
        eB = torch.cuda.Event(enable_timing=True)
        e0.record()
        chain(True, True)
        snap = outA.float().abs().sum()          # C: a plain launch reading all of A's out
        while not eB.query():                    # host polling: eB done must imply eA done
            pass
        if not eA.query():
            bad_host += 1
        torch.cuda.synchronize()
        if eA.elapsed_time(eB) < 0:
            bad_events += 1
        if float(snap) != float(outA.float().abs().sum()):
            bad_read += 1
        print(f"trial {t}: " + "  ".join(f"{m} {x:.3f} ms" for m, x in times.items())
              + f"  | overlap run: eA->eB {eA.elapsed_time(eB):+.4f} ms", flush=True)
    print(f"event order violations {bad_events}/{trials}, host-poll violations {bad_host}/{trials}, "
          f"plain launch read before A finished {bad_read}/{trials}")


if __name__ == "__main__":
    main()
