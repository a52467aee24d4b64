"""Calibration only (not part of the product or the bench): NVIDIA's own
sm_100 attention (cuDNN through torch SDPA) against this repo's kernel on
the same shapes and the same power-capped B200, each looped for a few
seconds so the board settles at its power-limited clock, with nvidia-smi
sampled during the loop.

    python scripts/calib_cudnn.py [seconds_per_case]
"""
import os
import statistics
import subprocess
import sys
import threading
import time

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def sampler(stop, rows):
    q = "clocks.sm,power.draw"
    while not stop.is_set():
        try:
            out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                  "-i", "0"], capture_output=True, text=True, timeout=5).stdout
            rows.append([float(x) for x in out.strip().split(",")])
        except Exception:
            pass
        time.sleep(0.2)


def timed(fn, secs):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    one = s.elapsed_time(e)
    n = max(2, int(secs * 1000 / max(one, 1e-3)))
    rows, stop = [], threading.Event()
    th = threading.Thread(target=sampler, args=(stop, rows), daemon=True)
    th.start()
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = s.elapsed_time(e) / n
    load = rows[len(rows) // 4:] or rows
    mhz = statistics.median(r[0] for r in load) if load else float("nan")
    w = statistics.median(r[1] for r in load) if load else float("nan")
    return ms, mhz, w


def main():
    from paper_2412_20501_b200 import kernels as K
    from torch.nn.attention import SDPBackend, sdpa_kernel
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 6.0
    cases = [("causal S=32768", 32768, 32768, 32, 128, True),
             ("full 8192x16384", 8192, 16384, 32, 128, False),
             ("causal S=131072", 131072, 131072, 32, 128, True)]
    for name, tq, tk, h, d, causal in cases:
        q = (torch.randn(tq, h, d, device="cuda") * 0.5).to(torch.bfloat16)
        k = (torch.randn(tk, h, d, device="cuda") * 0.5).to(torch.bfloat16)
        v = torch.randn(tk, h, d, device="cuda").to(torch.bfloat16)
        pairs = tq * (tq + 1) // 2 if causal else tq * tk
        fl = 4 * h * d * pairs
        out = torch.empty_like(q)
        lse = torch.empty(h, tq, device="cuda")
        ours = lambda: K.attention_block(q, k, v, 2 if causal else 0, 0, 0, out=out, lse=lse)  # noqa: E731
        # SDPA wants (B, H, S, D); the (S, H, D) buffers viewed as such are strided
        qt, kt, vt = (x.permute(1, 0, 2).unsqueeze(0) for x in (q, k, v))
        qc, kc, vc = (x.contiguous() for x in (qt, kt, vt))

        def cudnn(qq=qt, kk=kt, vv=vt):
            with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
                return F.scaled_dot_product_attention(qq, kk, vv, is_causal=causal)

        def cudnn_c():
            return cudnn(qc, kc, vc)
        for label, fn in (("ours", ours), ("cudnn (S,H,D) strided", cudnn),
                          ("cudnn (B,H,S,D) contiguous", cudnn_c), ("ours", ours)):
            try:
                ms, mhz, w = timed(fn, secs)
                print(f"{name:18s} {label:28s} {ms:9.3f} ms {fl / ms / 1e9:8.1f} TFLOP/s "
                      f"sm {mhz:6.0f} MHz {w:5.0f} W  {fl / ms / 1e9 / (mhz / 1000):6.1f} TF/GHz",
                      flush=True)
            except Exception as ex:  # calibration only
                print(f"{name:18s} {label:28s} failed: {type(ex).__name__}: {ex}", flush=True)
        if tq <= 32768:
            ref = cudnn_c().squeeze(0).permute(1, 0, 2).float()
            mine = ours()[0].float()
            print(f"{name:18s} max |ours - cudnn| = {(ref - mine).abs().max().item():.3e}", flush=True)
        del q, k, v, qc, kc, vc, out, lse
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
