"""Clock / power under sustained load (diagnostic, not the bench): runs one
workload back to back for a few seconds while sampling nvidia-smi, and
prints TFLOP/s next to the median SM clock and board power.

    python scripts/power_probe.py attn-full|attn-causal|gemm [seconds]
"""
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _ablib import maybe_use_env_library  # noqa: E402
maybe_use_env_library()


def sampler(stop, rows):
    q = "clocks.sm,power.draw,power.limit,clocks_throttle_reasons.active,temperature.gpu"
    while not stop.is_set():
        try:
            out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                  "-i", "0"], capture_output=True, text=True, timeout=5).stdout
            rows.append([x.strip() for x in out.strip().split(",")])
        except Exception:
            pass
        time.sleep(0.2)


def main():
    what = sys.argv[1]
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 6.0
    if what.startswith("attn"):
        from paper_2412_20501_b200 import kernels as K
        causal = what == "attn-causal"
        tq, tk = (32768, 32768) if causal else (8192, 16384)
        h, d = 32, 128
        q = torch.randn(tq, h, d, device="cuda").to(torch.bfloat16) * 0.5
        k = torch.randn(tk, h, d, device="cuda").to(torch.bfloat16) * 0.5
        v = torch.randn(tk, h, d, device="cuda").to(torch.bfloat16)
        out = torch.empty_like(q)
        lse = torch.empty(h, tq, device="cuda")
        fn = lambda: K.attention_block(q, k, v, 2 if causal else 0, 0, 0, out=out, lse=lse)  # noqa
        flops = 4 * h * d * (tq * (tq + 1) // 2 if causal else tq * tk)
    else:
        n = 8192
        a = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
        c = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
        fn = lambda: torch.matmul(a, b, out=c)  # noqa
        flops = 2 * n ** 3
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    stop, rows = threading.Event(), []
    th = threading.Thread(target=sampler, args=(stop, rows), daemon=True)
    th.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    iters = 0
    s.record()
    while time.time() - t0 < secs:
        for _ in range(5):
            fn()
        iters += 5
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = s.elapsed_time(e) / iters
    clk = sorted(float(r[0]) for r in rows[2:] if r and r[0].replace(".", "").isdigit())
    pw = sorted(float(r[1]) for r in rows[2:] if len(r) > 1 and r[1].replace(".", "").isdigit())
    med = lambda x: x[len(x) // 2] if x else float("nan")  # noqa
    print(f"{what:12s} {flops / ms / 1e9:8.1f} TFLOP/s  sm_clock_med {med(clk):6.0f} MHz  "
          f"power_med {med(pw):6.1f} W  limit {rows[-1][2] if rows else '?'} W  "
          f"reasons {sorted(set(r[3] for r in rows if len(r) > 3))}  temp {rows[-1][4] if rows else '?'}")


if __name__ == "__main__":
    main()
